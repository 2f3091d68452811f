// kmx_packcf.cu -- K1 for the carry-free packs as a STREAMING kernel: the
// value at 2^N (pack.py:79-84) or at 2^N of the reversed vector
// (pack_reversed, pack.py:87-93) of unsigned coefficients when N >= b, i.e.
// ks1 and ks2 (ksint.py:219-247): the coefficients do not overlap, so packed
// limb q is a pure function of the one or two coefficients (more when N < 32)
// whose bit ranges meet [32q, 32q + 32) -- no carries, no staging, no scans.
//
// One thread per four consecutive limbs (one 16-byte store); the coefficient
// words come straight from global memory (neighbouring threads read
// neighbouring words, L1/L2 serve the overlap), so the kernel moves
// in_words * 4 bytes in and ~N/8 bytes out per coefficient and is bound by
// HBM on long operands.  The range check rides on the top word of every
// coefficient a thread meets; the operand's bit length (meta, for MulStats) is
// a block max + one atomicMax per CTA.
//
// Used for large jobs (>= 2^20 packed limbs per call) and for multi-word
// coefficients on operands of >= 256 limbs; the block-per-operand kernels of
// kmx_pack.cu keep the rest, where their staged vectors win.
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

namespace {

constexpr int CF_T = 256;  // threads per CTA, 4 limbs each

// Coefficient cursor: position i (position order), its word pointer, and the
// step to the next position's words (+iw, or -iw for the reversed packs).
struct CfCur {
  const u32* p;   // words of coefficient i (undefined past L: guarded by i < L)
  int i, t;       // window start: bit t of coefficient i, 0 <= t < N
};

// BIAS (signed inputs, one word per coefficient): every loaded word is range-checked as a signed
// b-bit value and lifted by 2^(b-1) (the bias lift of the signed path); the prefix sums the
// correction needs are written by k_prefix_cf below.
template <int IW, bool SMALLN, bool BIAS = false>  // IW = 0: any in_words; SMALLN: N < 32 (several coefficients per limb)
__global__ void __launch_bounds__(CF_T) k_pack_cf(PackArgs A) {
  // grid: x = (pair, op), y = chunk of 4 * CF_T limbs
  const int job = blockIdx.x;
  const int pair = job / A.nops, o = job - pair * A.nops;
  const PackOp& P = A.op[o];
  const int mq = (P.m + 3) & ~3;  // the operand's row, rounded to whole 16-byte stores
  const int N = A.N, L = P.len;
  const int iw = IW ? IW : A.in_words;
  const bool rev = (P.kind & 2) != 0;
  const int step = rev ? -iw : iw;
  const u32* cf = P.coeffs + (long long)pair * P.coeff_pair_stride;
  const int topsh = (!BIAS && P.validate && (A.b & 31)) ? (A.b & 31) : 0;  // bits >= b of the top word must be zero
  bool bad = false;
  const u32 biasw = 1u << ((A.b - 1) & 31), bmask = A.b >= 32 ? 0xffffffffu : ((1u << A.b) - 1u);
  const bool vchk = BIAS && P.validate && A.b < 32;
  auto lift = [&](u32 raw) -> u32 {  // BIAS: signed range check + bias lift
    if (!BIAS) return raw;
    if (vchk) {
      const int v = (int)raw;
      bad |= v < -(1 << (A.b - 1)) || v >= (1 << (A.b - 1));
    }
    return (raw + biasw) & bmask;
  };
  const int q0 = 4 * (blockIdx.y * CF_T + threadIdx.x);
  u32 d[4] = {0u, 0u, 0u, 0u};
  if (q0 < mq) {
    const unsigned bit0 = 32u * (unsigned)q0;
    int i = (int)(bit0 / (unsigned)N);
    int t = (int)(bit0 - (unsigned)i * (unsigned)N);
    const u32* p = cf + (long long)(rev ? L - 1 - i : i) * iw;
    // one straight-line body per limb (both sides of a coefficient boundary in
    // the same instruction stream: a warp always straddles some boundary, so a
    // separate fast path would only add its instructions to the slow one's)
#pragma unroll
    for (int v = 0; v < 4; v++) {
      u32 x = 0u;
      if (i < L) {
        const int w = t >> 5;
        if (IW == 1) {
          const u32 lo = t < 32 ? lift(__ldg(p)) : 0u;
          if (topsh && t < 32) bad |= (lo >> topsh) != 0u;
          x = lo >> (t & 31);
        } else if (w < iw) {
          const u32 lo = __ldg(p + w);
          const u32 hi = w + 1 < iw ? __ldg(p + w + 1) : 0u;
          if (topsh) bad |= ((w == iw - 1 ? lo : (w + 2 == iw ? hi : 0u)) >> topsh) != 0u;
          x = __funnelshift_r(lo, hi, t & 31);
        }
        // coefficient(s) that start inside this window
        const int sh = N - t;
        if (SMALLN) {
          const u32* pn = p;
          for (int k = 1, s2 = sh; s2 < 32 && i + k < L; k++, s2 += N) {
            pn += step;
            const u32 lo = IW == 1 ? lift(__ldg(pn)) : __ldg(pn);
            if (topsh) bad |= (lo >> topsh) != 0u;
            x |= lo << s2;
          }
        } else if (sh < 32 && i + 1 < L) {
          const u32 lo = IW == 1 ? lift(__ldg(p + step)) : __ldg(p + step);
          if (topsh && iw == 1) bad |= (lo >> topsh) != 0u;
          x |= lo << sh;
        }
      }
      d[v] = x;
      t += 32;
      if (SMALLN) {
        while (t >= N) { t -= N; i++; p += step; }
      } else if (t >= N) {
        t -= N; i++; p += step;
      }
    }
    u32* out = P.out + (long long)pair * P.out_pair_stride;
    *reinterpret_cast<uint4*>(out + q0) = make_uint4(d[0], d[1], d[2], d[3]);
  }
  // bit length: block max, one atomic per CTA (meta zeroed before the launch)
  int top = 0;
#pragma unroll
  for (int v = 0; v < 4; v++)
    if (d[v]) top = 32 * (q0 + v) + 32 - __clz(d[v]);
  __shared__ int s_top[CF_T / 32];
  const unsigned wmax = __reduce_max_sync(0xffffffffu, (unsigned)top);
  if ((threadIdx.x & 31) == 0) s_top[threadIdx.x >> 5] = (int)wmax;
  const bool anybad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    int mx = 0;
    for (int w = 0; w < CF_T / 32; w++) mx = s_top[w] > mx ? s_top[w] : mx;
    if (mx) atomicMax(reinterpret_cast<int*>(P.meta + (long long)pair * P.meta_pair_stride + 1), mx);
    if (anybad) raise_err(A.err, ERR_INVAL);
  }
}

// Prefix sums of the lifted coefficients of one operand vector per CTA (signed path):
// out[0] = 0, out[i + 1] = sum_{k <= i} ((c_k + 2^(b-1)) mod 2^b).
__global__ void __launch_bounds__(256) k_prefix_cf(const u32* coeffs, long long coeff_pair_stride, int len, int b,
                                                   unsigned long long* prefix, long long prefix_pair_stride) {
  const long long pair = blockIdx.x;
  const u32 biasw = 1u << ((b - 1) & 31), bmask = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
  block_prefix_u64(coeffs + pair * coeff_pair_stride, len, biasw, bmask, prefix + pair * prefix_pair_stride);
}

}  // namespace

// Carry-free, every output row padded to 4 limbs and 16-byte aligned; unsigned inputs, or signed
// one-word inputs (bias lift in the kernel, prefix sums by k_prefix_cf).
bool pack_cf_ok(const PackArgs& a, int batch) {
  static const int force = getenv("KMX_PACK_CF") ? atoi(getenv("KMX_PACK_CF")) : -1;
  if (force == 0) return false;
  // signed inputs: opt-in (KMX_PACK_CF_SIGNED=1).  Measured at c2: the streaming pack plus its two
  // prefix-sum launches take 42.8 / 44.7 us (ks1 / ks2) against 35.4 / 39.2 us for the block kernel
  static const int cf_signed = getenv("KMX_PACK_CF_SIGNED") ? atoi(getenv("KMX_PACK_CF_SIGNED")) : 0;
  if (a.N < a.b || a.nops < 1 || batch < 1) return false;
  if (a.bias && (!cf_signed || a.in_words != 1 || a.b < 1 || a.b > 32)) return false;
  long long limbs = 0;
  for (int i = 0; i < a.nops; i++) {
    const PackOp& p = a.op[i];
    if ((p.kind & 1) || (p.prefix && !a.bias)) return false;
    if ((reinterpret_cast<uintptr_t>(p.out) & 15) || (p.out_pair_stride & 3)) return false;
    if (p.out_pair_stride < ((p.m + 3) & ~3)) return false;  // room for the rounding limbs
    if ((long long)p.len * a.N + 64 >= (1LL << 31) || p.m > 65535LL * 4 * CF_T) return false;
    limbs += (long long)batch * p.m;
  }
  // meta of all ops of a pair is one contiguous block starting at op[0].meta
  for (int i = 0; i < a.nops; i++)
    if (a.op[i].meta_pair_stride != a.op[0].meta_pair_stride || a.op[i].meta < a.op[0].meta ||
        a.op[i].meta - a.op[0].meta >= a.op[0].meta_pair_stride)
      return false;
  // measured (config-5 sweep with KMX_PACK_CF=0 / 1): large calls always; small ones only with
  // multi-word coefficients on operands of >= 256 limbs (3-10% faster; one-word or short: 3-25% slower)
  if (a.bias) return force == 1 || limbs >= (1LL << 19);
  return force == 1 || limbs >= (1LL << 20) || (a.in_words >= 2 && a.op[0].m >= 256 && a.op[0].len >= 64);
}

cudaError_t launch_pack_cf(const PackArgs& a, int batch, cudaStream_t st) {
  // meta = [sign 0, bit length 0] before the atomics
  cudaError_t e = cudaMemsetAsync(a.op[0].meta, 0, (size_t)batch * a.op[0].meta_pair_stride * sizeof(u32), st);
  if (e != cudaSuccess) return e;
  int mmax = 0;
  for (int i = 0; i < a.nops; i++) mmax = a.op[i].m > mmax ? a.op[i].m : mmax;
  const int mq = (mmax + 3) & ~3;
  // (f and g operands may differ in m: the grid covers the larger, each CTA bounds by its own)
  dim3 grid(batch * a.nops, (mq / 4 + CF_T - 1) / CF_T);
  if (grid.y > 65535) return cudaErrorInvalidValue;
  if (a.bias) {
    if (a.N < 32) k_pack_cf<1, true, true><<<grid, CF_T, 0, st>>>(a);
    else k_pack_cf<1, false, true><<<grid, CF_T, 0, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    for (int i = 0; i < a.nops; i++) {
      const PackOp& p = a.op[i];
      if (!p.prefix) continue;
      k_prefix_cf<<<batch, 256, 0, st>>>(p.coeffs, p.coeff_pair_stride, p.len, a.b, p.prefix, p.prefix_pair_stride);
    }
    return cudaGetLastError();
  }
  if (a.N < 32) {
    if (a.in_words == 1) k_pack_cf<1, true><<<grid, CF_T, 0, st>>>(a);
    else k_pack_cf<0, true><<<grid, CF_T, 0, st>>>(a);
  } else {
    switch (a.in_words) {
      case 1: k_pack_cf<1, false><<<grid, CF_T, 0, st>>>(a); break;
      case 2: k_pack_cf<2, false><<<grid, CF_T, 0, st>>>(a); break;
      case 4: k_pack_cf<4, false><<<grid, CF_T, 0, st>>>(a); break;
      case 8: k_pack_cf<8, false><<<grid, CF_T, 0, st>>>(a); break;
      default: k_pack_cf<0, false><<<grid, CF_T, 0, st>>>(a); break;
    }
  }
  return cudaGetLastError();
}

}  // namespace kmx
