// Shared device primitives for the KS kernels (sm_100a).
//
// Carry resolution.  Every stage of the path ends in the same problem: a run
// of 32-bit digit positions each holding a small signed 64-bit value y_q, and
// we want the normalized digits of V = sum y_q 2^(32q).  We split
// y = lo + 2^32 hi (hi small), shift hi one position up (z_q = lo_q + hi_{q-1}),
// after which every carry lies in {-1, 0, +1}.  The carry out of a digit is
// then a function of the carry into it, c_out = floor((z + c_in) / 2^32), i.e.
// a map {-1,0,1} -> {-1,0,1}, stored in 6 bits.  Maps compose associatively,
// so a warp/block prefix scan over maps resolves every carry chain in
// O(log n) steps regardless of propagate runs (no data-dependent loops).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kmx {

typedef uint32_t u32;
typedef uint64_t u64;
typedef int64_t i64;

// error bits latched in the workspace flag word
enum : u32 { ERR_INVAL = 1u, ERR_RECON = 2u, ERR_INEXACT = 4u };

__device__ __forceinline__ void raise_err(u32* flag, u32 bit) { atomicOr(flag, bit); }

// ---------------------------------------------------------------- carry maps
// entry i (i = c_in + 1) holds c_out + 1 in bits [2i, 2i+2)
constexpr u32 CM_IDENT = 0x24u;  // 0->0, 1->1, 2->2

__device__ __forceinline__ u32 cm_make(i64 z) {
  u32 m = 0;
#pragma unroll
  for (int c = -1; c <= 1; c++) {
    i64 o = (z + c) >> 32;  // arithmetic shift: floor division
    m |= (u32)(o + 1) << (2 * (c + 1));
  }
  return m;
}
// x -> g(f(x))
__device__ __forceinline__ u32 cm_compose(u32 f, u32 g) {
  u32 r = 0;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    u32 fi = (f >> (2 * i)) & 3u;
    r |= ((g >> (2 * fi)) & 3u) << (2 * i);
  }
  return r;
}
__device__ __forceinline__ int cm_apply(u32 m, int c) { return (int)((m >> (2 * (c + 1))) & 3u) - 1; }

// Segmented exclusive scan of carry maps over segments of G consecutive
// threads (G a power of two dividing blockDim.x, or G == blockDim.x).
// Returns the exclusive prefix for this thread; *total receives the
// inclusive map of the whole segment.  `sm` needs blockDim.x/32 words.
// Must be called by all threads of the block.
__device__ __forceinline__ u32 cm_seg_scan(u32 m, int G, u32* sm, u32* total) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int w = G < 32 ? G : 32;
  const int sl = lane & (w - 1);
  u32 inc = m;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    if (off < w) {
      u32 o = __shfl_up_sync(0xffffffffu, inc, off, w);
      if (sl >= off) inc = cm_compose(o, inc);
    }
  }
  u32 exc = __shfl_up_sync(0xffffffffu, inc, 1, w);
  if (sl == 0) exc = CM_IDENT;
  if (G <= 32) {
    *total = __shfl_sync(0xffffffffu, inc, w - 1, w);
    return exc;
  }
  // segments spanning several warps
  const int wps = G >> 5;  // warps per segment
  __syncthreads();
  if (lane == 31) sm[warp] = inc;
  __syncthreads();
  const int w0 = (warp / wps) * wps;
  u32 pre = CM_IDENT;
  for (int k = w0; k < warp; k++) pre = cm_compose(pre, sm[k]);
  u32 tot = pre;
  for (int k = warp; k < w0 + wps; k++) tot = cm_compose(tot, sm[k]);
  *total = tot;
  __syncthreads();
  return cm_compose(pre, exc);
}

// ------------------------------------------------------ multiply-accumulate
// 96-bit column accumulator += a*b.  ptxas fuses the pair into one
// IMAD.WIDE.U32 with a carry-out predicate, and two consecutive addc into a
// single IADD3.X absorbing both carries (checked in SASS).
__device__ __forceinline__ void mac96(u32& c0, u32& c1, u32& c2, u32 a, u32 b) {
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
      "addc.u32 %2, %2, 0;"
      : "+r"(c0), "+r"(c1), "+r"(c2)
      : "r"(a), "r"(b));
}

__host__ __device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ long long cdivll(long long a, long long b) { return (a + b - 1) / b; }

// Block prefix sums (signed inputs' bias lift; used by K1 and the bias kernel).
static __device__ void block_prefix_u64(const u32* x, int n, u32 bias, u32 bmask, unsigned long long* out) {
  // out[0] = 0, out[i+1] = sum_{k<=i} ((x[k] + bias) & bmask)
  __shared__ unsigned long long wsum[8];
  __shared__ unsigned long long run;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { run = 0; out[0] = 0; }
  __syncthreads();
  for (int i0 = 0; i0 < n; i0 += blockDim.x) {
    const int i = i0 + tid;
    unsigned long long v = i < n ? (unsigned long long)((x[i] + bias) & bmask) : 0ull;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v += o;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    unsigned long long pre = run;
    for (int k = 0; k < warp; k++) pre += wsum[k];
    if (i < n) out[i + 1] = pre + v;
    __syncthreads();
    if (tid == blockDim.x - 1) run = pre + v;
    __syncthreads();
  }
}

// Read 32 bits starting at bit `bit` of a little-endian word array of
// `nwords` words (bits beyond the array read as zero).
__device__ __forceinline__ u32 bits32(const u32* w, int nwords, long long bit) {
  if (bit < 0) {
    if (bit <= -32) return 0u;
    u32 x = (nwords > 0) ? w[0] : 0u;
    return x << (int)(-bit);
  }
  long long q = bit >> 5;
  int s = (int)(bit & 31);
  u32 lo = q < nwords ? w[q] : 0u;
  if (s == 0) return lo;
  u32 hi = (q + 1) < nwords ? w[q + 1] : 0u;
  return (lo >> s) | (hi << (32 - s));
}

}  // namespace kmx
