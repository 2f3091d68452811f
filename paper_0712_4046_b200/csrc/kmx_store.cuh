// kmx_store.cuh -- coefficient stores shared by the finish and
// reconstruction kernels (kmx_ks.cu, kmx_finish.cu).
#pragma once

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

// ---- signed-input bias correction applied at store time (see BiasFix)
__device__ __forceinline__ void store_coeff128(u32* dst, int ow, unsigned __int128 hp, long long k, const BiasFix& bf,
                                               long long pair) {
  u64 lo = (u64)hp, hi = (u64)(hp >> 64);
  if (bf.enabled) {
    const unsigned long long* PF = bf.pf + pair * bf.pair_stride;
    // coefficient indices < 2^31: 32-bit index arithmetic
    const int kk = (int)k, lf = bf.lf, lg = bf.lg, lgp = bf.lgpad;
    const int i0 = max(kk - lg + 1, 0), i1 = min(kk, lf - 1);
    const int j0 = max(kk - lf + 1, 0), j1 = min(kk, lg - 1);
    // staged copies (lgpad >= 0) live in shared memory, padded: entry i at
    // i + (i >> lgpad) (PG follows PF); read them with ld.shared
    const u32 sbase = lgp >= 0 ? (u32)__cvta_generic_to_shared(PF) : 0u;
    auto pe = [&](int i) -> u64 {
      if (lgp < 0) return __ldg(PF + i);  // read-only for the kernel: loads may move above the stores
      u64 v;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sbase + 8u * (u32)(i + (i >> lgp))));
      return v;
    };
    const int g0 = lf + 1;
    const u64 S = (pe(i1 + 1) - pe(i0)) + (pe(g0 + j1 + 1) - pe(g0 + j0));
    const u64 cnt = (u64)(i1 - i0 + 1);
    const int sh1 = bf.b - 1, sh2 = 2 * bf.b - 2;       // 0..31, 0..62
    const u64 a_lo = S << sh1, a_hi = sh1 ? (S >> (64 - sh1)) : 0ull;
    const u64 c_lo = cnt << sh2, c_hi = sh2 ? (cnt >> (64 - sh2)) : 0ull;
    const u64 l1 = lo - a_lo;                          // v - S 2^(b-1)
    const u64 h1 = hi - a_hi - (l1 > lo ? 1ull : 0ull);
    lo = l1 + c_lo;                                    // + cnt 2^(2b-2)
    hi = h1 + c_hi + (lo < l1 ? 1ull : 0ull);
  }
  const u32 ext = (hi >> 63) ? 0xffffffffu : 0u;
  if (ow == 3) {  // 12-byte records (c2): one 8-byte and one 4-byte store
    if ((reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
      *reinterpret_cast<uint2*>(dst) = make_uint2((u32)lo, (u32)(lo >> 32));
      dst[2] = (u32)hi;
    } else {
      dst[0] = (u32)lo;
      *reinterpret_cast<uint2*>(dst + 1) = make_uint2((u32)(lo >> 32), (u32)hi);
    }
    return;
  }
  dst[0] = (u32)lo;
  if (ow > 1) dst[1] = (u32)(lo >> 32);
  if (ow > 2) dst[2] = (u32)hi;
  if (ow > 3) dst[3] = (u32)(hi >> 32);
  for (int w = 4; w < ow; w++) dst[w] = ext;
}

}  // namespace kmx
