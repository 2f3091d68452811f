// kmx_packseg.cu -- K1 for long operands and small batches: every pack op
// split into 2048-limb segments, one CTA each, so a batch of a few dozen
// pairs (BASELINE config 4: 32 pairs, operands of 8578..34300 limbs) fills
// the chip instead of running one CTA per operand.  Same values as pack_op
// (kmx_pack.cuh; pack.py:62-110): E + O 2^N, or |E - O 2^N| with the larger
// stream first, from the unstaged coefficient vectors.
//
//   k_pseg_pre  one warp per (pair, op): the top-down order of E and O 2^N
//               for the negated packs, the sign word of the meta, a cleared
//               bit length, and the signed path's prefix sums;
//   k_pseg_a    one CTA per (pair, op, segment): the range check of a slice
//               of the coefficients (pack.py:36-46), the segment's digits
//               with carry-in 0 (thread carry maps + one block scan) and its
//               segment carry map;
//   k_pseg_b    one CTA per (pair, op, segment): the segment's carry-in from
//               the maps before it, rippled through the (rare) run of
//               propagating digits, and the top nonzero digit (bit length).
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"
#include "kmx_pack.cuh"

namespace kmx {

namespace {

constexpr int PS_T = 256;
constexpr int PS_SEG = PS_T * PK_V;  // limbs per segment

struct SegArgs {
  PackArgs pk;
  int nseg;       // segments of the longest op
  int* order;     // [pair][op]: +1 E first, -1 O first
  u32* maps;      // [pair][op][seg] segment carry maps (cm_ encoding)
};

__device__ __forceinline__ PackCtx<false> seg_ctx(const PackArgs& A, int pair, int o) {
  PackCtx<false> C;
  C.cf = A.op[o].coeffs + (long long)pair * A.op[o].coeff_pair_stride;
  C.sc = nullptr;
  C.L = A.op[o].len;
  C.N = A.N;
  C.b = A.b;
  C.iw = A.in_words;
  C.rev = (A.op[o].kind & 2) != 0;
  C.bias = A.bias != 0;
  C.bmask = C.b >= 32 ? 0xffffffffu : ((1u << C.b) - 1u);
  C.biasw = A.bias ? (1u << (C.b - 1)) : 0u;
  return C;
}

__global__ void __launch_bounds__(128) k_pseg_pre(SegArgs sa, int nitems) {
  const PackArgs& A = sa.pk;
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (item >= nitems) return;
  const int pair = item / A.nops, o = item - pair * A.nops;
  const PackOp& P = A.op[o];
  const PackCtx<false> C = seg_ctx(A, pair, o);
  if (P.prefix) {  // signed path: prefix sums of the lifted coefficients, natural order
    unsigned long long* out = P.prefix + (long long)pair * P.prefix_pair_stride;
    unsigned long long run = 0ull;
    if (lane == 0) out[0] = 0ull;
    for (int i0 = 0; i0 < C.L; i0 += 32) {
      const int i = i0 + lane;
      unsigned long long inc = i < C.L ? (unsigned long long)((__ldg(C.cf + (long long)i * C.iw) + C.biasw) & C.bmask) : 0ull;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
      }
      if (i < C.L) out[i + 1] = run + inc;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  const int S = 2 * C.N, m = P.m;
  int order = 1;
  if (P.kind & 1) {
    int ord = 0;
    for (int base = m - 1; base >= 0 && ord == 0; base -= 32) {
      const int q = base - lane;
      u32 e = 0u, ov = 0u;
      if (q >= 0) {
        StreamCur ce, co;
        ce.init(q, 0, S);
        co.init(q, C.N, S);
        e = ce.bits(C, 0, S);
        ov = co.bits(C, 1, S);
      }
      const unsigned diff = __ballot_sync(0xffffffffu, e != ov);
      if (diff) ord = __shfl_sync(0xffffffffu, e > ov ? 1 : -1, __ffs(diff) - 1);
    }
    order = ord >= 0 ? 1 : -1;
  }
  if (lane == 0) {
    sa.order[item] = order;
    const bool flip = P.kind == 3 && (C.L & 1) == 0;  // pack.py:106-109
    u32* meta = P.meta + (long long)pair * P.meta_pair_stride;
    meta[0] = (P.kind & 1) ? (((order < 0) != flip) ? 1u : 0u) : 0u;
    meta[1] = 0u;  // k_pseg_b takes the max over the segments
  }
}

__global__ void __launch_bounds__(PS_T) k_pseg_a(SegArgs sa) {
  __shared__ u32 sm_scan[PS_T / 32];
  const PackArgs& A = sa.pk;
  const int item = blockIdx.x / sa.nseg, seg = blockIdx.x - item * sa.nseg;
  const int pair = item / A.nops, o = item - pair * A.nops;
  const PackOp& P = A.op[o];
  const int m = P.m;
  if (seg * PS_SEG >= m) return;  // shorter op: no such segment (uniform across the block)
  const PackCtx<false> C = seg_ctx(A, pair, o);
  if (P.validate) {  // range check (pack.py:36-46): this segment's slice of the coefficient words
    const int nseg_op = (m + PS_SEG - 1) / PS_SEG;
    const long long nw = (long long)C.L * C.iw;
    const long long w0 = nw * seg / nseg_op, w1 = nw * (seg + 1) / nseg_op;
    bool bad = false;
    for (long long x = w0 + threadIdx.x; x < w1; x += PS_T) {
      const u32 raw = __ldg(C.cf + x);
      if (A.bias) {
        const int v = (int)raw;
        if (C.b < 32) bad |= (v < -(1 << (C.b - 1))) || (v >= (1 << (C.b - 1)));
      } else {
        const int lo_bit = 32 * (int)(x % C.iw);
        if (lo_bit >= C.b) bad |= raw != 0u;
        else if (C.b - lo_bit < 32) bad |= (raw >> (C.b - lo_bit)) != 0u;
      }
    }
    if (bad) raise_err(A.err, ERR_INVAL);
  }
  const bool neg = P.kind & 1;
  const int order = sa.order[item];
  const int S = 2 * C.N;
  const int q0 = seg * PS_SEG + threadIdx.x * PK_V;
  StreamCur ce, co;
  ce.init(q0, 0, S);
  co.init(q0, C.N, S);
  u32 d[PK_V];
  int c = 0;
  u32 allF = 0xffffffffu, any = 0u;
#pragma unroll
  for (int v = 0; v < PK_V; v++) {
    u32 e = 0u, ov = 0u;
    if (q0 + v < m) {
      e = ce.bits(C, 0, S);
      ov = co.bits(C, 1, S);
    }
    ce.next(S);
    co.next(S);
    const i64 x = (!neg ? (i64)e + ov : (order > 0 ? (i64)e - ov : (i64)ov - e)) + c;
    d[v] = (u32)x;
    c = (int)(x >> 32);
    allF &= d[v];
    any |= d[v];
  }
  const u32 M = (u32)(c - (any == 0u ? 1 : 0) + 1) | ((u32)(c + 1) << 2) |
                ((u32)(c + (allF == 0xffffffffu ? 1 : 0) + 1) << 4);
  u32 tot;
  const u32 exc = cm_seg_scan(M, PS_T, sm_scan, &tot);
  int k = cm_apply(exc, 0);
  if (k) {
#pragma unroll
    for (int v = 0; v < PK_V; v++) {
      const u32 old = d[v];
      d[v] = old + (u32)k;
      k = k > 0 ? (d[v] == 0u ? 1 : 0) : (k < 0 && old == 0u ? -1 : 0);
    }
  }
  u32* out = P.out + (long long)pair * P.out_pair_stride;
  if (q0 + PK_V <= m) {
    uint4* dst = reinterpret_cast<uint4*>(out + q0);
    dst[0] = make_uint4(d[0], d[1], d[2], d[3]);
    dst[1] = make_uint4(d[4], d[5], d[6], d[7]);
  } else {
#pragma unroll
    for (int v = 0; v < PK_V; v++)
      if (q0 + v < m) out[q0 + v] = d[v];
  }
  if (threadIdx.x == 0) sa.maps[(long long)item * sa.nseg + seg] = tot;
}

__global__ void __launch_bounds__(PS_T) k_pseg_b(SegArgs sa) {
  __shared__ int sm_cin, sm_first;
  __shared__ unsigned long long sm_top;
  const PackArgs& A = sa.pk;
  const int item = blockIdx.x / sa.nseg, seg = blockIdx.x - item * sa.nseg;
  const int pair = item / A.nops, o = item - pair * A.nops;
  const PackOp& P = A.op[o];
  const int m = P.m;
  const int nseg_op = (m + PS_SEG - 1) / PS_SEG;
  if (seg >= nseg_op) return;
  if (threadIdx.x == 0) {
    const u32* mp = sa.maps + (long long)item * sa.nseg;
    int c = 0;
    for (int k = 0; k < seg; k++) c = cm_apply(mp[k], c);
    sm_cin = c;
    sm_first = PS_T;
    sm_top = 0ull;
    // the operand fits in m limbs: no carry out of its top segment
    if (seg == nseg_op - 1 && cm_apply(mp[seg], c) != 0) raise_err(A.err, ERR_INEXACT);
  }
  __syncthreads();
  const int cin = sm_cin;
  u32* out = P.out + (long long)pair * P.out_pair_stride;
  const int q0 = seg * PS_SEG + threadIdx.x * PK_V;
  u32 d[PK_V];
#pragma unroll
  for (int v = 0; v < PK_V; v++) d[v] = q0 + v < m ? out[q0 + v] : 0u;
  if (cin) {
    // carry +1 runs through all-ones digits, a borrow through all-zero ones
    const u32 prop = cin > 0 ? 0xffffffffu : 0u;
    bool all = true;
#pragma unroll
    for (int v = 0; v < PK_V; v++) all &= (q0 + v >= m) || d[v] == prop;
    if (!all) atomicMin(&sm_first, (int)threadIdx.x);
    __syncthreads();
    const int first = sm_first;
    if ((int)threadIdx.x <= first) {
      int k = cin;
#pragma unroll
      for (int v = 0; v < PK_V; v++) {
        if (q0 + v >= m || !k) break;
        const u32 old = d[v];
        d[v] = old + (u32)k;
        k = k > 0 ? (d[v] == 0u ? 1 : 0) : (old == 0u ? -1 : 0);
        out[q0 + v] = d[v];
      }
    }
  }
  int top = 0;
  u32 topv = 0u;
#pragma unroll
  for (int v = 0; v < PK_V; v++)
    if (q0 + v < m && d[v]) { top = q0 + v + 1; topv = d[v]; }
  const unsigned wmax = __reduce_max_sync(0xffffffffu, (unsigned)top);
  if (wmax) {
    const int src = __ffs(__ballot_sync(0xffffffffu, (unsigned)top == wmax)) - 1;
    const u32 v = __shfl_sync(0xffffffffu, topv, src);
    if ((threadIdx.x & 31) == 0) atomicMax(&sm_top, ((unsigned long long)wmax << 32) | v);
  }
  __syncthreads();
  if (threadIdx.x == 0 && sm_top) {
    const int t = (int)(sm_top >> 32);
    u32* meta = P.meta + (long long)pair * P.meta_pair_stride;
    atomicMax(&meta[1], (u32)(32 * (t - 1) + 32 - __clz((u32)sm_top)));
  }
}

}  // namespace

size_t pack_seg_scratch_bytes(int batch, int nops, int mmax) {
  const int nseg = (mmax + PS_SEG - 1) / PS_SEG;
  return (((size_t)batch * nops * 4 + 255) & ~(size_t)255) + (size_t)batch * nops * nseg * 4;
}

// Segmented pack: long operands and too few (pair, op) blocks to fill the
// chip with the block-per-operand kernel (KMX_PACK_SEG=1 / 0 forces on / off).
bool pack_seg_wanted(const PackArgs& a, int batch) {
  static const int force = getenv("KMX_PACK_SEG") ? atoi(getenv("KMX_PACK_SEG")) : -1;
  if (!a.scratch || force == 0) return false;
  int mmax = 0;
  for (int i = 0; i < a.nops; i++) mmax = a.op[i].m > mmax ? a.op[i].m : mmax;
  if (a.scratch_bytes < pack_seg_scratch_bytes(batch, a.nops, mmax)) return false;
  if (force == 1) return true;
  // measured at c4 (32 pairs): ks1 / ks2 / ks3 pack 144 / 76 / 87 -> 67 / 66 /
  // 66 us; ks4 (256 operands of 8578 limbs) stays faster unsegmented (58 us)
  return mmax >= 2 * PS_SEG && (long long)batch * a.nops < 148;
}

cudaError_t launch_pack_seg(const PackArgs& a, int batch, cudaStream_t st) {
  int mmax = 0;
  for (int i = 0; i < a.nops; i++) mmax = a.op[i].m > mmax ? a.op[i].m : mmax;
  SegArgs sa;
  sa.pk = a;
  sa.nseg = (mmax + PS_SEG - 1) / PS_SEG;
  const int nitems = batch * a.nops;
  sa.order = reinterpret_cast<int*>(a.scratch);
  sa.maps = reinterpret_cast<u32*>(reinterpret_cast<char*>(a.scratch) + (((size_t)nitems * 4 + 255) & ~(size_t)255));
  if (nitems == 0) return cudaSuccess;
  k_pseg_pre<<<(nitems + 3) / 4, 128, 0, st>>>(sa, nitems);
  k_pseg_a<<<nitems * sa.nseg, PS_T, 0, st>>>(sa);
  k_pseg_b<<<nitems * sa.nseg, PS_T, 0, st>>>(sa);
  return cudaGetLastError();
}

}  // namespace kmx
