// kmx_pack.cu -- K1, the standalone pack kernel: evaluation of the
// coefficient vectors at +-2^N, +-2^-N (pack.py:62-110, bignat._pack_ints
// bignat.py:411-428), one block per (pair, pack op); the per-operand body is
// pack_op in kmx_pack.cuh (shared with the fused tensor-core prologue).
#include <cstdio>
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"
#include "kmx_pack.cuh"

namespace kmx {

template <bool STAGED>
__global__ void __launch_bounds__(PK_T) k_pack(PackArgs A) {
  extern __shared__ u32 pk_sc[];
  const int pair = blockIdx.x / A.nops;
  pack_op<STAGED>(A, pair, blockIdx.x - pair * A.nops, pk_sc, nullptr);
}

// ops (2q, 2q+1) = (pack, pack_negated) or (pack_reversed, pack_negated_reversed)
__global__ void __launch_bounds__(PK_T) k_pack_pair(PackArgs A) {
  extern __shared__ u32 pk_sc[];
  const int npairs = A.nops / 2;
  const int pair = blockIdx.x / npairs;
  const int q = blockIdx.x - pair * npairs;
  pack_pair(A, pair, 2 * q, 2 * q + 1, pk_sc);
}

static bool pairable(const PackArgs& a) {
  if (a.nops < 4 || (a.nops & 1)) return false;
  for (int q = 0; 2 * q + 1 < a.nops; q++) {
    const PackOp &x = a.op[2 * q], &y = a.op[2 * q + 1];
    if ((x.kind & 1) || y.kind != (x.kind | 1) || x.coeffs != y.coeffs || x.len != y.len ||
        x.coeff_pair_stride != y.coeff_pair_stride)
      return false;
  }
  return true;
}

bool pack_w1_ok(const PackArgs& a);
bool pack_seg_wanted(const PackArgs& a, int batch);
cudaError_t launch_pack_seg(const PackArgs& a, int batch, cudaStream_t st);
cudaError_t launch_pack_w1(const PackArgs& a, int batch, bool paired, cudaStream_t st);
bool pack_cf_ok(const PackArgs& a, int batch);
cudaError_t launch_pack_cf(const PackArgs& a, int batch, cudaStream_t st);

cudaError_t launch_pack(const PackArgs& a, int batch, cudaStream_t st) {
  static const int use_pair = getenv("KMX_PACK_PAIR") ? atoi(getenv("KMX_PACK_PAIR")) : 1;
  // large carry-free unsigned packs (ks1 / ks2): the streaming kernel (kmx_packcf.cu)
  if (pack_cf_ok(a, batch)) return launch_pack_cf(a, batch, st);
  // long operands, small batches: segments of every operand on separate CTAs
  if (pack_seg_wanted(a, batch)) return launch_pack_seg(a, batch, st);
  // one-word coefficients at 2N >= 32, + and - operands from one staged vector
  // (ks3 / ks4) up to 1024 limbs: the warp-per-job kernel (kmx_pack1.cu).
  // Measured at c2: ks4 pack 48.8 -> 38.0 us, ks3 37 -> 37.5 us (m = 1184);
  // single-operand jobs with long operands (ks1 / ks2, m = 2367 / 1184) are
  // faster on the block kernel below (35 / 38 us vs 56 / 49 us).
  {
    int mmax0 = 0;
    for (int i = 0; i < a.nops; i++) mmax0 = a.op[i].m > mmax0 ? a.op[i].m : mmax0;
    static const int w1_force = getenv("KMX_PACK_W1") ? atoi(getenv("KMX_PACK_W1")) : -1;
    const bool paired = use_pair && pairable(a);
    // one-word coefficients read through the streaming accumulator (Str1): the
    // warp kernel also wins on longer paired jobs (c2 ks3, m = 1184: pack 37.5 ->
    // 30.1 us).  Single jobs stay on the block kernel: the warp kernel is 5-15%
    // slower there at small n (config-5 sweep) and at m = 2367 (c2 ks1 35.0 vs 40.1)
    const bool w1_auto = paired && mmax0 <= (a.in_words == 1 ? 2048 : 1024);
    if (pack_w1_ok(a) && (w1_force == 1 || w1_auto))
      return launch_pack_w1(a, batch, paired, st);
  }
  int mmax = 0;
  for (int i = 0; i < a.nops; i++) mmax = a.op[i].m > mmax ? a.op[i].m : mmax;
  int T = ((mmax + PK_V - 1) / PK_V + 31) & ~31;  // sized to the operand
  if (T < 32) T = 32;
  if (T > PK_T) T = PK_T;
  int lmax = 0;
  for (int i = 0; i < a.nops; i++) lmax = a.op[i].len > lmax ? a.op[i].len : lmax;
  PackArgs b = a;
  static const int fast = getenv("KMX_PACK_FAST") ? atoi(getenv("KMX_PACK_FAST")) : 1;
  b.fast1 = fast;
  const int nw = (lmax + PK_PAD) * a.in_words;
  // The carry-free pack (no negated op, N >= b) stages vectors up to 80 KB of
  // opt-in shared memory (unstaged windows cost two global loads each):
  // config 5 n=4096 b=128 ks1 / ks2 pack 158 / 107 -> 76 / 89 us, n=8192 b=64
  // ks2 84 -> 50 us.  Larger stages (1 CTA per SM) and the carry paths (ks3 /
  // ks4: 125 -> 151 us at n=4096 b=128) measured slower: they keep 48 KB.
  bool carry_free = a.N >= a.b;
  for (int i = 0; i < a.nops; i++) carry_free &= (a.op[i].kind & 1) == 0;
  static const int big = getenv("KMX_PACK_STAGE_WORDS") ? atoi(getenv("KMX_PACK_STAGE_WORDS")) : 20480;
  b.stage = nw <= (carry_free ? big : PK_STAGE_WORDS);
  const size_t smem = b.stage ? (size_t)nw * sizeof(u32) : 0;
  // paired packs halve the block count: only when that still fills the chip
  // (c1, 64 pairs: 256 paired blocks are slower than 512 single ones)
  if (b.stage && use_pair && pairable(a) && (use_pair > 1 || (long long)batch * (a.nops / 2) >= 148LL * 8)) {
    if (smem > 44 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k_pack_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_pack_pair<<<batch * (a.nops / 2), T, smem, st>>>(b);
    return cudaGetLastError();
  }
  if (getenv("KMX_DEBUG_PACK"))
    fprintf(stderr, "launch_pack: batch=%d nops=%d T=%d stage=%d smem=%zu N=%d b=%d iw=%d m=%d\n", batch, a.nops, T,
            b.stage, smem, a.N, a.b, a.in_words, mmax);
  if (b.stage) {
    if (smem > 44 * 1024) {  // + static shared memory must fit the opt-in limit
      cudaError_t e = cudaFuncSetAttribute(k_pack<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_pack<true><<<batch * a.nops, T, smem, st>>>(b);
  } else {
    k_pack<false><<<batch * a.nops, T, 0, st>>>(b);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && getenv("KMX_DEBUG_PACK")) fprintf(stderr, "launch_pack: %s\n", cudaGetErrorString(e));
  return e;
}

}  // namespace kmx
