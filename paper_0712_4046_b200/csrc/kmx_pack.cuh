// kmx_pack.cuh -- K1, the pack of one operand (pack.py:55-110), shared by the
// standalone pack kernel (kmx_ks.cu, operands to global memory for the
// integer-pipe multiply) and the tensor-core multiply (kmx_tc.cu), which
// packs its two operands straight into shared memory.
#pragma once

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

// ========================================================================
// K1: pack.  One block per (pair, operand) (or per product when fused).  The packed value is
// V = sum_i s_i d_i 2^(iN) (d_i = c_i, or c_(L-1-i) for the reversed packs;
// s_i = (-1)^i for the negated packs, times -1 for pack_negated_reversed at
// even L, pack.py:62-110).  Because 2N >= b (pack.py:55-59) the even- and
// odd-position coefficients each form a clean bitstream E, O, so digit q of
// V is e_q + o_q (positive packs, carries in {0,1}) or |e_q - o_q| with the
// larger stream first (negated packs; the order is decided up front by a
// top-down warp compare of E and O, so the magnitude is produced in one pass
// -- sign-magnitude as SignedBig, bignat.py:218-277).  Each thread owns
// PK_V consecutive digits and walks the coefficient windows incrementally;
// carries are resolved with one block scan of carry maps per chunk.
// ========================================================================
// Prefix sums of n staged values in natural order (x[i] at x[rev ? n-1-i : i]):
// out[0] = 0, out[i+1] = sum_{k<=i} x[k].  Each thread owns a contiguous
// segment; one block scan of the segment sums.
static __device__ void block_prefix_staged(const u32* x, int n, bool rev, unsigned long long* out) {
  __shared__ unsigned long long wsum[32];
  const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg = (n + T - 1) / T;
  const int a = min(n, tid * seg), e = min(n, a + seg);
  unsigned long long s = 0ull;
  for (int i = a; i < e; i++) s += x[rev ? n - 1 - i : i];
  unsigned long long v = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, v, off);
    if (lane >= off) v += o;
  }
  if (lane == 31) wsum[warp] = v;
  __syncthreads();
  unsigned long long run = v - s;
  for (int k = 0; k < warp; k++) run += wsum[k];
  if (tid == 0) out[0] = 0ull;
  for (int i = a; i < e; i++) {
    run += x[rev ? n - 1 - i : i];
    out[i + 1] = run;
  }
  __syncthreads();
}

constexpr int PK_T = 256;
constexpr int PK_V = 8;

template <bool STAGED>
struct PackCtx {
  const u32* cf;
  const u32* sc;   // staged coefficients in position order (reversal and bias applied)
  int L, N, b, iw;
  bool rev, bias;
  u32 biasw, bmask;
  __device__ __forceinline__ u32 word(int i, int w) const {  // word w of the coefficient at position i
    if (STAGED) return w < iw ? sc[i * iw + w] : 0u;  // zero-padded past L (staged)
    return gword(i, w);
  }
  __device__ __forceinline__ u32 gword(int i, int w) const {  // unstaged (very long vectors)
    if (i >= L || w >= iw) return 0u;
    const int ci = rev ? (L - 1 - i) : i;
    u32 x = __ldg(cf + (long long)ci * iw + w);
    if (bias) x = (x + biasw) & bmask;  // signed inputs: lift by 2^(b-1) (iw == 1)
    return x;
  }
};
constexpr int PK_STAGE_WORDS = 12288;  // stage coefficient vectors up to 48 KB
constexpr int PK_PAD = 64;             // zero positions past L (window reads beyond the top)

// Cursor over one parity stream: coefficients at positions i = 2m + par start
// at bit off + m*S (S = 2N >= b, so they never overlap inside a stream).
// Invariant for the current digit q: m = the last coefficient starting at or
// below bit 32q (m may be -1), t = 32q - start(m).
struct StreamCur {
  int m, t;
  __device__ __forceinline__ void init(int q, int off, int S) {
    const int x = 32 * q - off;
    m = x >= 0 ? x / S : -((-x + S - 1) / S);
    t = x - m * S;
  }
  __device__ __forceinline__ void next(int S) {
    t += 32;
    while (t >= S) { t -= S; m++; }
  }
  // spacing S >= 32 (and S >= b, as always): at most the tail of coefficient
  // m and the head of coefficient m+1 meet a 32-bit window, so no loops
  // (staged vectors are zero-padded past L; bits at or above b are zero)
  __device__ __forceinline__ void next1(int S) {
    t += 32;
    if (t >= S) { t -= S; m++; }
  }
  template <class Ctx>
  __device__ __forceinline__ u32 bits1(const Ctx& C, int par, int S) const {  // one-word coefficients
    u32 v = (m >= 0 && t < C.b) ? (C.sc[2 * m + par] >> t) : 0u;
    const int sh = S - t;
    if (sh < 32) v |= C.sc[2 * (m + 1) + par] << sh;
    return v;
  }
  template <class Ctx>
  __device__ __forceinline__ u32 bitsw(const Ctx& C, int par, int S) const {  // multi-word coefficients
    u32 v = 0u;
    if (m >= 0 && t < C.b) {
      const int wq = t >> 5;
      const u32* p = C.sc + (2 * m + par) * C.iw + wq;
      v = __funnelshift_r(p[0], wq + 1 < C.iw ? p[1] : 0u, t & 31);
    }
    const int sh = S - t;
    if (sh < 32) v |= C.sc[(2 * (m + 1) + par) * C.iw] << sh;
    return v;
  }
  // the 32 bits of this stream in the current digit window
  template <class Ctx>
  __device__ __forceinline__ u32 bits(const Ctx& C, int par, int S) const {
    u32 v = 0u;
    if (m >= 0 && t < C.b) {
      const int wq = t >> 5, sb = t & 31;
      const int i = 2 * m + par;
      const u32 lo = C.word(i, wq);
      v = sb ? ((lo >> sb) | (C.word(i, wq + 1) << (32 - sb))) : lo;
    }
    for (int k = 1, sh = S - t; sh < 32; k++, sh += S) {  // coefficients starting inside the window
      if (m + k >= 0) v |= C.word(2 * (m + k) + par, 0) << sh;
    }
    return v;
  }
};

// One packed operand (pack op o of pair `pair`) into `out` (global or shared
// memory), its [sign, bitlen] meta, and -- on the ops that carry them -- the
// range check and the signed prefix sums.  Called by every thread of the
// block (block-wide barriers); pk_sc: (len + PK_PAD) * in_words words of
// shared memory for the staged vector.  out == nullptr: the op's own
// global operand slot.  side_effects = false skips the meta, prefix and range
// check writes (another block of the same product does them).
template <bool STAGED>
__device__ __forceinline__ void pack_op(const PackArgs& A, int pair, int o, u32* pk_sc, u32* out_override,
                                        bool side_effects = true) {
  __shared__ u32 sm_scan[PK_T / 32];
  __shared__ int sm_order, sm_bad;
  __shared__ unsigned long long sm_top;  // (top nonzero digit index + 1) << 32 | its value
  const int T = blockDim.x;  // 32..PK_T, sized to the operand
  __shared__ i64 sm_carry;
  const int tid = threadIdx.x;
  PackCtx<STAGED> C;
  C.cf = A.op[o].coeffs + (long long)pair * A.op[o].coeff_pair_stride;
  u32* out = out_override ? out_override : A.op[o].out + (long long)pair * A.op[o].out_pair_stride;
  u32* meta = A.op[o].meta + (long long)pair * A.op[o].meta_pair_stride;
  const int kind = A.op[o].kind, m = A.op[o].m;
  C.L = A.op[o].len; C.N = A.N; C.b = A.b; C.iw = A.in_words;
  C.rev = (kind & 2) != 0;
  C.bias = A.bias != 0;
  C.bmask = C.b >= 32 ? 0xffffffffu : ((1u << C.b) - 1u);
  C.biasw = A.bias ? (1u << (C.b - 1)) : 0u;
  const bool neg = kind & 1;
  const bool flip = (kind == 3) && ((C.L & 1) == 0);  // pack.py:106-109
  const bool validate = side_effects && A.op[o].validate != 0;
  unsigned long long* prefix = side_effects ? A.op[o].prefix : nullptr;
  C.sc = pk_sc;
  if (tid == 0) sm_bad = 0;
  if (STAGED) {
    // stage the vector in position order with zero padding: every load of
    // the CTA in flight at once, the range check (pack.py:36-46) on the raw
    // words, then the bias lift and the reversal
    const int L = C.L, iw = C.iw, nw = L * iw;
    __syncthreads();
    bool bad = false;
    auto put = [&](int x, u32 raw) {
      const int i = iw == 1 ? x : x / iw, w = iw == 1 ? 0 : x - i * iw;
      if (validate) {
        if (C.bias) {
          const int v = (int)raw;
          if (C.b < 32) bad |= (v < -(1 << (C.b - 1))) || (v >= (1 << (C.b - 1)));
        } else {
          const int lo_bit = 32 * w;
          if (lo_bit >= C.b) bad |= raw != 0u;
          else if (C.b - lo_bit < 32) bad |= (raw >> (C.b - lo_bit)) != 0u;
        }
      }
      const u32 v = C.bias ? ((raw + C.biasw) & C.bmask) : raw;
      const int p = C.rev ? L - 1 - i : i;
      pk_sc[p * iw + w] = v;
    };
    if ((nw & 3) == 0 && (reinterpret_cast<uintptr_t>(C.cf) & 15) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(C.cf);
#pragma unroll 4
      for (int x4 = tid; x4 < nw / 4; x4 += T) {
        const uint4 r = __ldg(s4 + x4);
        put(4 * x4, r.x);
        put(4 * x4 + 1, r.y);
        put(4 * x4 + 2, r.z);
        put(4 * x4 + 3, r.w);
      }
    } else {
#pragma unroll 4
      for (int x = tid; x < nw; x += T) put(x, __ldg(C.cf + x));
    }
    for (int x = nw + tid; x < (L + PK_PAD) * iw; x += T) pk_sc[x] = 0u;
    if (bad) sm_bad = 1;
    __syncthreads();
    if (tid == 0 && sm_bad) raise_err(A.err, ERR_INVAL);
    if (prefix)  // signed path: prefix sums of the lifted coefficients (iw == 1)
      block_prefix_staged(pk_sc, L, C.rev, prefix + (long long)pair * A.op[o].prefix_pair_stride);
  } else {
    if (validate) {  // CoeffVec invariant 0 <= c < 2^b (pack.py:36-46)
      for (int i = tid; i < C.L; i += T) {
        const u32* c = C.cf + (long long)i * C.iw;
        bool bad = false;
        if (A.bias) {
          const int v = (int)c[0];
          if (C.b < 32) bad = (v < -(1 << (C.b - 1))) || (v >= (1 << (C.b - 1)));
        } else {
          for (int w = 0; w < C.iw; w++) {
            const int lo_bit = 32 * w;
            if (lo_bit >= C.b) bad |= c[w] != 0u;
            else if (C.b - lo_bit < 32) bad |= (c[w] >> (C.b - lo_bit)) != 0u;
          }
        }
        if (bad) raise_err(A.err, ERR_INVAL);
      }
    }
    if (prefix) {  // signed path: prefix sums of the lifted coefficients
      block_prefix_u64(C.cf, C.L, C.biasw, C.bmask, prefix + (long long)pair * A.op[o].prefix_pair_stride);
      __syncthreads();
    }
  }
  if (tid == 0) { sm_top = 0ull; sm_order = 1; sm_carry = 0; }
  const int S = 2 * C.N;
  // negated packs: order of E and O from the most significant differing digit
  if (neg && tid < 32) {
    int order = 0;  // +1: E > O, -1: E < O, 0: equal
    for (int base = m - 1; base >= 0 && order == 0; base -= 32) {
      const int q = base - tid;
      u32 e = 0u, ov = 0u;
      if (q >= 0) {
        StreamCur ce, co;
        ce.init(q, 0, S);
        co.init(q, C.N, S);
        e = ce.bits(C, 0, S);
        ov = co.bits(C, 1, S);
      }
      const unsigned diff = __ballot_sync(0xffffffffu, e != ov);
      if (diff) {
        const int l = __ffs(diff) - 1;  // lowest lane = highest digit
        const int gt = __shfl_sync(0xffffffffu, e > ov ? 1 : 0, l);
        order = gt ? 1 : -1;
      }
    }
    if (tid == 0) sm_order = order >= 0 ? 1 : -1;
  }
  __syncthreads();
  const int order = sm_order;  // E - O (order 1) or O - E (order -1)
  const int negative = neg ? ((order < 0) != flip ? 1 : 0) : 0;

  int my_top = 0;
  u32 my_topv = 0u;
  // loop-free windows: every width in the carry-free disjoint path; one-word
  // coefficients only in the carry path (multi-word there measured slower:
  // c1 ks3/ks4 pack 19 -> 21 us)
  const bool fastw = STAGED && A.fast1 && S >= 32 && C.b <= S;
  const bool fast1 = fastw && C.iw == 1;
  if (!neg && C.N >= C.b && fastw) {
    for (int q0 = tid * PK_V; q0 < m; q0 += T * PK_V) {
      StreamCur ce, co;
      ce.init(q0, 0, S);
      co.init(q0, C.N, S);
#pragma unroll 1
      for (int v = 0; v < PK_V && q0 + v < m; v++) {
        const u32 d = fast1 ? (ce.bits1(C, 0, S) | co.bits1(C, 1, S)) : (ce.bitsw(C, 0, S) | co.bitsw(C, 1, S));
        ce.next1(S);
        co.next1(S);
        out[q0 + v] = d;
        if (d) { my_top = q0 + v + 1; my_topv = d; }
      }
    }
  } else if (!neg && C.N >= C.b) {
    // disjoint bit fields (pack.py:66-67): V = E | O, no carries at all --
    // a pure gather, every thread independent
    for (int q0 = tid * PK_V; q0 < m; q0 += T * PK_V) {
      StreamCur ce, co;
      ce.init(q0, 0, S);
      co.init(q0, C.N, S);
#pragma unroll 1
      for (int v = 0; v < PK_V && q0 + v < m; v++) {
        const u32 d = ce.bits(C, 0, S) | co.bits(C, 1, S);
        ce.next(S);
        co.next(S);
        out[q0 + v] = d;
        if (d) { my_top = q0 + v + 1; my_topv = d; }
      }
    }
  } else
  for (int c0 = 0; c0 < m; c0 += T * PK_V) {
    const int q0 = c0 + tid * PK_V;
    StreamCur ce, co;
    ce.init(q0, 0, S);
    co.init(q0, C.N, S);
    // t_v = e_v +- o_v lies in (-2^32, 2^33), so carries stay in {-1, 0, 1}.
    // Resolve this thread's digits with carry-in 0; a carry-in of +1 (-1)
    // alters the carry-out only when those digits are all ones (all zeros),
    // so the thread's carry map is (c0 - all0, c0, c0 + allF).
    u32 d[PK_V];
    int c = 0;
    u32 allF = 0xffffffffu, any = 0u;
#pragma unroll
    for (int v = 0; v < PK_V; v++) {
      const int q = q0 + v;
      u32 e = 0u, ov = 0u;
      if (fast1) {
        if (q < m) {
          e = ce.bits1(C, 0, S);
          ov = co.bits1(C, 1, S);
        }
        ce.next1(S);
        co.next1(S);
      } else {
        if (q < m) {
          e = ce.bits(C, 0, S);
          ov = co.bits(C, 1, S);
        }
        ce.next(S);
        co.next(S);
      }
      const i64 x = (!neg ? (i64)e + ov : (order > 0 ? (i64)e - ov : (i64)ov - e)) + c;
      d[v] = (u32)x;
      c = (int)(x >> 32);
      allF &= d[v];
      any |= d[v];
    }
    const u32 M = (u32)(c - (any == 0u ? 1 : 0) + 1) | ((u32)(c + 1) << 2) |
                  ((u32)(c + (allF == 0xffffffffu ? 1 : 0) + 1) << 4);
    u32 tot;
    const u32 exc = cm_seg_scan(M, T, sm_scan, &tot);
    const int cin = (int)sm_carry;
    int k = cm_apply(exc, cin);
    if (k) {  // ripple the carry-in through this thread's digits
#pragma unroll
      for (int v = 0; v < PK_V; v++) {
        const u32 old = d[v];
        d[v] = old + (u32)k;
        k = k > 0 ? (d[v] == 0u ? 1 : 0) : (k < 0 && old == 0u ? -1 : 0);
      }
    }
#pragma unroll
    for (int v = 0; v < PK_V; v++)
      if (q0 + v < m && d[v]) { my_top = q0 + v + 1; my_topv = d[v]; }
    if (q0 + PK_V <= m) {
      uint4* dst = reinterpret_cast<uint4*>(out + q0);
      dst[0] = make_uint4(d[0], d[1], d[2], d[3]);
      dst[1] = make_uint4(d[4], d[5], d[6], d[7]);
    } else {
#pragma unroll
      for (int v = 0; v < PK_V; v++)
        if (q0 + v < m) out[q0 + v] = d[v];
    }
    __syncthreads();
    if (tid == 0) sm_carry = cm_apply(tot, cin);
    __syncthreads();
  }
  if (tid == 0 && sm_carry != 0) raise_err(A.err, ERR_INEXACT);  // operand overflow (cannot happen)
  {  // top nonzero digit: warp max first, one shared atomic per warp
    const unsigned wmax = __reduce_max_sync(0xffffffffu, (unsigned)my_top);
    if (wmax) {
      const int src = __ffs(__ballot_sync(0xffffffffu, (unsigned)my_top == wmax)) - 1;
      const u32 v = __shfl_sync(0xffffffffu, my_topv, src);
      if ((tid & 31) == 0) atomicMax(&sm_top, ((unsigned long long)wmax << 32) | v);
    }
  }
  __syncthreads();
  if (tid == 0 && side_effects) {
    const int top = (int)(sm_top >> 32);
    meta[0] = (u32)negative;
    meta[1] = top ? (u32)(32 * (top - 1) + 32 - __clz((u32)sm_top)) : 0u;
  }
}

// ------------------------------------------------------------------------
// pack_pair: the two packs that share a coefficient order -- value at +2^N
// and at -2^N (ops o0: kind 0 or 2, o1: kind 1 or 3; pack.py:79-110) -- from
// ONE staged copy of the vector: the even / odd bitstreams E, O are extracted
// once per digit and feed both E + O (carries {0,1}) and |E - O| (sign from
// the top-down warp compare), each with its own thread-level carry maps and
// block scan.  Staged vectors only (the caller checks the size).
// ------------------------------------------------------------------------
__device__ __forceinline__ void pack_pair(const PackArgs& A, int pair, int o0, int o1, u32* pk_sc) {
  __shared__ u32 sm_scan[2][PK_T / 32];
  __shared__ int sm_order, sm_bad;
  __shared__ unsigned long long sm_top[2];
  __shared__ i64 sm_carry[2];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  PackCtx<true> C;
  const PackOp& P0 = A.op[o0];
  const PackOp& P1 = A.op[o1];
  C.cf = P0.coeffs + (long long)pair * P0.coeff_pair_stride;
  u32* out0 = P0.out + (long long)pair * P0.out_pair_stride;
  u32* out1 = P1.out + (long long)pair * P1.out_pair_stride;
  const int m = P0.m > P1.m ? P0.m : P1.m;
  C.L = P0.len; C.N = A.N; C.b = A.b; C.iw = A.in_words;
  C.rev = (P0.kind & 2) != 0;
  C.bias = A.bias != 0;
  C.bmask = C.b >= 32 ? 0xffffffffu : ((1u << C.b) - 1u);
  C.biasw = A.bias ? (1u << (C.b - 1)) : 0u;
  const bool flip = (P1.kind == 3) && ((C.L & 1) == 0);  // pack.py:106-109
  const bool validate = P0.validate != 0 || P1.validate != 0;
  unsigned long long* prefix = P0.prefix ? P0.prefix : P1.prefix;
  const long long pstride = P0.prefix ? P0.prefix_pair_stride : P1.prefix_pair_stride;
  C.sc = pk_sc;
  if (tid == 0) sm_bad = 0;
  {
    const int L = C.L, iw = C.iw, nw = L * iw;
    __syncthreads();
    bool bad = false;
    auto put = [&](int x, u32 raw) {
      const int i = iw == 1 ? x : x / iw, w = iw == 1 ? 0 : x - i * iw;
      if (validate) {
        if (C.bias) {
          const int v = (int)raw;
          if (C.b < 32) bad |= (v < -(1 << (C.b - 1))) || (v >= (1 << (C.b - 1)));
        } else {
          const int lo_bit = 32 * w;
          if (lo_bit >= C.b) bad |= raw != 0u;
          else if (C.b - lo_bit < 32) bad |= (raw >> (C.b - lo_bit)) != 0u;
        }
      }
      const u32 v = C.bias ? ((raw + C.biasw) & C.bmask) : raw;
      const int p = C.rev ? L - 1 - i : i;
      pk_sc[p * iw + w] = v;
    };
    if ((nw & 3) == 0 && (reinterpret_cast<uintptr_t>(C.cf) & 15) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(C.cf);
#pragma unroll 4
      for (int x4 = tid; x4 < nw / 4; x4 += T) {
        const uint4 r = __ldg(s4 + x4);
        put(4 * x4, r.x);
        put(4 * x4 + 1, r.y);
        put(4 * x4 + 2, r.z);
        put(4 * x4 + 3, r.w);
      }
    } else {
#pragma unroll 4
      for (int x = tid; x < nw; x += T) put(x, __ldg(C.cf + x));
    }
    for (int x = nw + tid; x < (L + PK_PAD) * iw; x += T) pk_sc[x] = 0u;
    if (bad) sm_bad = 1;
    __syncthreads();
    if (tid == 0 && sm_bad) raise_err(A.err, ERR_INVAL);
    if (prefix) block_prefix_staged(pk_sc, L, C.rev, prefix + (long long)pair * pstride);
  }
  if (tid == 0) { sm_top[0] = sm_top[1] = 0ull; sm_order = 1; sm_carry[0] = sm_carry[1] = 0; }
  const int S = 2 * C.N;
  if (tid < 32) {  // order of E and O from the most significant differing digit
    int order = 0;
    for (int base = m - 1; base >= 0 && order == 0; base -= 32) {
      const int q = base - tid;
      u32 e = 0u, ov = 0u;
      if (q >= 0) {
        StreamCur ce, co;
        ce.init(q, 0, S);
        co.init(q, C.N, S);
        e = ce.bits(C, 0, S);
        ov = co.bits(C, 1, S);
      }
      const unsigned diff = __ballot_sync(0xffffffffu, e != ov);
      if (diff) {
        const int l = __ffs(diff) - 1;
        const int gt = __shfl_sync(0xffffffffu, e > ov ? 1 : 0, l);
        order = gt ? 1 : -1;
      }
    }
    if (tid == 0) sm_order = order >= 0 ? 1 : -1;
  }
  __syncthreads();
  const int order = sm_order;
  const int negative = (order < 0) != flip ? 1 : 0;
  int top0 = 0, top1 = 0;
  u32 topv0 = 0u, topv1 = 0u;
  // loop-free windows for one-word coefficients only: with multi-word
  // coefficients (c1, b = 64) the extra loop variant costs this kernel more
  // than it saves (c1 ks3/ks4 pack 19 -> 21 us); pack_op takes them
  const bool fast1 = A.fast1 && S >= 32 && C.b <= S && C.iw == 1;
  for (int c0 = 0; c0 < m; c0 += T * PK_V) {
    const int q0 = c0 + tid * PK_V;
    StreamCur ce, co;
    ce.init(q0, 0, S);
    co.init(q0, C.N, S);
    u32 d0[PK_V], d1[PK_V];
    int k0 = 0, k1 = 0;
    u32 f0 = 0xffffffffu, a0 = 0u, f1 = 0xffffffffu, a1 = 0u;
    auto digit = [&](int v, u32 e, u32 ov) {
      const i64 x0 = (i64)e + ov + k0;
      const i64 x1 = (order > 0 ? (i64)e - ov : (i64)ov - e) + k1;
      d0[v] = (u32)x0;
      k0 = (int)(x0 >> 32);
      d1[v] = (u32)x1;
      k1 = (int)(x1 >> 32);
      f0 &= d0[v]; a0 |= d0[v];
      f1 &= d1[v]; a1 |= d1[v];
    };
    if (fast1) {
#pragma unroll
      for (int v = 0; v < PK_V; v++) {
        u32 e = 0u, ov = 0u;
        if (q0 + v < m) {
          e = ce.bits1(C, 0, S);
          ov = co.bits1(C, 1, S);
        }
        ce.next1(S);
        co.next1(S);
        digit(v, e, ov);
      }
    } else {
#pragma unroll
      for (int v = 0; v < PK_V; v++) {
        u32 e = 0u, ov = 0u;
        if (q0 + v < m) {
          e = ce.bits(C, 0, S);
          ov = co.bits(C, 1, S);
        }
        ce.next(S);
        co.next(S);
        digit(v, e, ov);
      }
    }
    // thread carry maps (c0 - all0, c0, c0 + allF), one block scan per stream
    const u32 M0 = (u32)(k0 - (a0 == 0u ? 1 : 0) + 1) | ((u32)(k0 + 1) << 2) |
                   ((u32)(k0 + (f0 == 0xffffffffu ? 1 : 0) + 1) << 4);
    const u32 M1 = (u32)(k1 - (a1 == 0u ? 1 : 0) + 1) | ((u32)(k1 + 1) << 2) |
                   ((u32)(k1 + (f1 == 0xffffffffu ? 1 : 0) + 1) << 4);
    u32 tot0, tot1;
    const u32 e0 = cm_seg_scan(M0, T, sm_scan[0], &tot0);
    const u32 e1 = cm_seg_scan(M1, T, sm_scan[1], &tot1);
    const int cin0 = (int)sm_carry[0], cin1 = (int)sm_carry[1];
    int r0 = cm_apply(e0, cin0), r1 = cm_apply(e1, cin1);
    if (r0) {
#pragma unroll
      for (int v = 0; v < PK_V; v++) {
        const u32 old = d0[v];
        d0[v] = old + (u32)r0;
        r0 = r0 > 0 ? (d0[v] == 0u ? 1 : 0) : (r0 < 0 && old == 0u ? -1 : 0);
      }
    }
    if (r1) {
#pragma unroll
      for (int v = 0; v < PK_V; v++) {
        const u32 old = d1[v];
        d1[v] = old + (u32)r1;
        r1 = r1 > 0 ? (d1[v] == 0u ? 1 : 0) : (r1 < 0 && old == 0u ? -1 : 0);
      }
    }
#pragma unroll
    for (int v = 0; v < PK_V; v++) {
      if (q0 + v < P0.m && d0[v]) { top0 = q0 + v + 1; topv0 = d0[v]; }
      if (q0 + v < P1.m && d1[v]) { top1 = q0 + v + 1; topv1 = d1[v]; }
    }
    if (q0 + PK_V <= P0.m) {
      uint4* dst = reinterpret_cast<uint4*>(out0 + q0);
      dst[0] = make_uint4(d0[0], d0[1], d0[2], d0[3]);
      dst[1] = make_uint4(d0[4], d0[5], d0[6], d0[7]);
    } else {
#pragma unroll
      for (int v = 0; v < PK_V; v++)
        if (q0 + v < P0.m) out0[q0 + v] = d0[v];
    }
    if (q0 + PK_V <= P1.m) {
      uint4* dst = reinterpret_cast<uint4*>(out1 + q0);
      dst[0] = make_uint4(d1[0], d1[1], d1[2], d1[3]);
      dst[1] = make_uint4(d1[4], d1[5], d1[6], d1[7]);
    } else {
#pragma unroll
      for (int v = 0; v < PK_V; v++)
        if (q0 + v < P1.m) out1[q0 + v] = d1[v];
    }
    __syncthreads();
    if (tid == 0) {
      sm_carry[0] = cm_apply(tot0, cin0);
      sm_carry[1] = cm_apply(tot1, cin1);
    }
    __syncthreads();
  }
  if (tid == 0 && (sm_carry[0] != 0 || sm_carry[1] != 0)) raise_err(A.err, ERR_INEXACT);
  {
    const unsigned w0 = __reduce_max_sync(0xffffffffu, (unsigned)top0);
    const unsigned w1 = __reduce_max_sync(0xffffffffu, (unsigned)top1);
    const u32 v0 = __shfl_sync(0xffffffffu, topv0, w0 ? __ffs(__ballot_sync(0xffffffffu, (unsigned)top0 == w0)) - 1 : 0);
    const u32 v1 = __shfl_sync(0xffffffffu, topv1, w1 ? __ffs(__ballot_sync(0xffffffffu, (unsigned)top1 == w1)) - 1 : 0);
    if ((tid & 31) == 0) {
      if (w0) atomicMax(&sm_top[0], ((unsigned long long)w0 << 32) | v0);
      if (w1) atomicMax(&sm_top[1], ((unsigned long long)w1 << 32) | v1);
    }
  }
  __syncthreads();
  if (tid == 0) {
    u32* meta0 = P0.meta + (long long)pair * P0.meta_pair_stride;
    u32* meta1 = P1.meta + (long long)pair * P1.meta_pair_stride;
    const int t0 = (int)(sm_top[0] >> 32), t1 = (int)(sm_top[1] >> 32);
    meta0[0] = 0u;
    meta0[1] = t0 ? (u32)(32 * (t0 - 1) + 32 - __clz((u32)sm_top[0])) : 0u;
    meta1[0] = (u32)negative;
    meta1[1] = t1 ? (u32)(32 * (t1 - 1) + 32 - __clz((u32)sm_top[1])) : 0u;
  }
}

}  // namespace kmx
