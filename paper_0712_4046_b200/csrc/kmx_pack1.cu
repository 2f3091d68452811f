// kmx_pack1.cu -- K1 for one- and two-word coefficients (b <= 64, in_words <= 2)
// at a parity spacing 2N >= 32: one WARP per pack job, no block barriers.
//
// Same values as pack_op / pack_pair (kmx_pack.cuh; pack.py:62-110): the
// value at +2^N, -2^N (and the reversed forms) of a coefficient vector, as
// the even / odd bitstreams E, O (spacing 2N, so each 32-bit window meets at
// most the tail of one coefficient and the head of the next) combined into
// E + O 2^N (carries {0, 1}) and |E - O 2^N| (borrows {-1, 0}, larger stream
// first, the order from a top-down compare).  A job is one (pair, op) or --
// for ks3 / ks4 -- one (pair, coefficient order) producing both the + and the
// - operand from one staged copy of the vector.
//
// Per job the warp stages the vector in shared memory (16-byte loads, range
// check, bias lift, reversal; the signed path's prefix sums by a warp scan),
// then walks the operand in 256-limb chunks: each lane resolves 8 digits per
// stream with carry-in 0 and a 2-bit carry map, one 5-step shuffle scan per
// stream composes the maps, the chunk's carry-in is a warp-uniform scalar,
// and every lane writes its 8 digits as two 16-byte stores.  This replaces
// the block-per-job kernel's barriers and block scans; it is the path for
// the headline shape (BASELINE config 2: N = 74 / 37 / 19 bits).
#include <cstdio>
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

namespace {

constexpr int W1_WARPS = 4;
constexpr int W1_V = 8;              // digits per lane per chunk
constexpr int W1_CH = 32 * W1_V;     // digits per chunk
constexpr int W1_PAD = 64;           // zero words past L (windows read beyond the top)

// Cursor over one parity stream (coefficients 2j + par start at bit off + j S)
struct Cur1 {
  int m, t;
  __device__ __forceinline__ void init(int q, int off, int S) {
    const int x = 32 * q - off;
    m = x >= 0 ? x / S : -((-x + S - 1) / S);
    t = x - m * S;
  }
  __device__ __forceinline__ void next(int S) {
    t += 32;
    if (t >= S) { t -= S; m++; }
  }
  // 32 bits of the stream at the current window (S >= 32, b <= S), for
  // coefficients of IW words (staged with one zero word of slack per vector)
  template <int IW>
  __device__ __forceinline__ u32 bits(const u32* sc, int par, int S, int b) const {
    u32 v = 0u;
    if (m >= 0 && t < b) {
      if (IW == 1) {
        v = sc[2 * m + par] >> t;
      } else {
        const u32* c = sc + (2 * m + par) * IW + (t >> 5);
        const u32 hi = (t >> 5) + 1 < IW ? c[1] : 0u;
        v = __funnelshift_r(c[0], hi, t & 31);
      }
    }
    const int sh = S - t;
    if (sh < 32) v |= sc[(2 * (m + 1) + par) * IW] << sh;
    return v;
  }
};

// Streaming reader of one parity stream of one-word coefficients (S >= 32,
// b <= 32): a 64-bit accumulator holds the stream from the current limb's
// first bit; `filled` is where the next coefficient starts.  One compare,
// and at most one load + 64-bit shift / or, per digit -- against a window
// extraction (two loads, two shifts, index arithmetic) per digit with the
// cursor above.
struct Str1 {
  unsigned long long acc;
  int filled, idx;
  __device__ __forceinline__ void init(int q, int off, int S, int par, const u32* sc) {
    const int x = 32 * q - off;  // >= -off > -S
    const int m = x >= 0 ? x / S : -1;
    const int t = x - m * S;     // bits into coefficient m (0 <= t < S)
    const u32 c = m >= 0 ? sc[2 * m + par] : 0u;
    acc = t < 32 ? (unsigned long long)(c >> t) : 0ull;
    filled = S - t;
    idx = 2 * (m + 1) + par;
  }
  __device__ __forceinline__ u32 next(int S, const u32* sc) {
    if (filled < 32) {
      acc |= (unsigned long long)sc[idx] << filled;
      idx += 2;
      filled += S;
    }
    const u32 d = (u32)acc;
    acc >>= 32;
    filled -= 32;
    return d;
  }
};

// {0,1}-carry map of a lane's digits: bit0 = carry out for carry-in 0,
// bit1 = for carry-in 1 (kmx_tcutil.cuh cm2 encoding); compose(later, earlier)
__device__ __forceinline__ u32 cmp2(u32 later, u32 earlier) {
  const u32 h0 = (later >> (earlier & 1u)) & 1u;
  const u32 h1 = (later >> ((earlier >> 1) & 1u)) & 1u;
  return h0 | (h1 << 1);
}

struct StreamAcc {  // the running top nonzero digit of one output stream
  int top;
  u32 topv;
};

template <int IW>
__global__ void __launch_bounds__(32 * W1_WARPS, 8) k_pack_w1(PackArgs A, int paired, int njobs, int psplit) {
  extern __shared__ u32 w1_sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int job = blockIdx.x * (blockDim.x >> 5) + warp;
  if (job >= njobs) return;
  const int per_pair = paired ? A.nops / 2 : A.nops;
  const int pair = job / per_pair;
  const int jq = job - pair * per_pair;
  const int o_pos = paired ? 2 * jq : ((A.op[jq].kind & 1) ? -1 : jq);
  const int o_neg = paired ? 2 * jq + 1 : ((A.op[jq].kind & 1) ? jq : -1);
  const PackOp& P = A.op[paired ? 2 * jq : jq];
  const int L = P.len, N = A.N, b = A.b, S = 2 * N;
  const bool rev = (P.kind & 2) != 0;
  const bool bias = A.bias != 0;
  const u32 bmask = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
  const u32 biasw = bias ? (1u << (b - 1)) : 0u;
  const bool validate = (o_pos >= 0 && A.op[o_pos].validate) || (o_neg >= 0 && A.op[o_neg].validate);
  const int m = P.m;
  u32* sc = w1_sm + warp * (L + W1_PAD) * IW;
  const u32* cf = P.coeffs + (long long)pair * P.coeff_pair_stride;

  // ---- stage: range check on the raw words, bias lift, reversal
  bool bad = false;
  auto put = [&](int x, u32 raw) {  // word x of the vector (coefficient x / IW)
    const int i = IW == 1 ? x : x / IW, w = IW == 1 ? 0 : x - i * IW;
    if (validate) {
      if (bias) {
        const int v = (int)raw;
        if (b < 32) bad |= (v < -(1 << (b - 1))) || (v >= (1 << (b - 1)));
      } else {
        const int lo_bit = 32 * w;
        if (lo_bit >= b) bad |= raw != 0u;
        else if (b - lo_bit < 32) bad |= (raw >> (b - lo_bit)) != 0u;
      }
    }
    sc[(rev ? L - 1 - i : i) * IW + w] = bias ? ((raw + biasw) & bmask) : raw;
  };
  const int nw = L * IW;
  if ((nw & 3) == 0 && (reinterpret_cast<uintptr_t>(cf) & 15) == 0) {
    // every load of a batch in flight before any is used (one warp stages the
    // whole vector: memory-level parallelism comes from the batch)
    const uint4* s4 = reinterpret_cast<const uint4*>(cf);
    const int n4 = nw / 4;
    for (int base = 0; base < n4; base += 32 * 8) {
      uint4 r[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int x4 = base + 32 * k + lane;
        r[k] = x4 < n4 ? __ldg(s4 + x4) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int x4 = base + 32 * k + lane;
        if (x4 < n4) {
          put(4 * x4, r[k].x);
          put(4 * x4 + 1, r[k].y);
          put(4 * x4 + 2, r[k].z);
          put(4 * x4 + 3, r[k].w);
        }
      }
    }
  } else {
    for (int x = lane; x < nw; x += 32) put(x, __ldg(cf + x));
  }
  for (int x = nw + lane; x < (L + W1_PAD) * IW; x += 32) sc[x] = 0u;
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_err(A.err, ERR_INVAL);
  __syncwarp();
  // ---- signed path: prefix sums of the lifted coefficients in natural order
  const PackOp* PP = (o_pos >= 0 && A.op[o_pos].prefix) ? &A.op[o_pos] : nullptr;
  if (PP) {  // coalesced: 32 consecutive entries per step, warp scan + running total
    unsigned long long* out = PP->prefix + (long long)pair * PP->prefix_pair_stride;
    unsigned long long run = 0ull;
    // psplit: the polynomial's forward job writes the entries of [0, h), its reversed job (which has
    // staged the same coefficients) those of [h, L) on top of the sum of the first h -- the scan is
    // ~1300 instructions on the jobs that carry it, so the two jobs of a polynomial share it
    int ibeg = 0, iend = L;
    if (psplit) {
      const int h = ((L >> 1) + 31) & ~31;
      if (rev) {
        ibeg = h;
        unsigned long long t = 0ull;
        for (int i = lane; i < h; i += 32) t += sc[(L - 1 - i) * IW];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
        run = t;
      } else {
        iend = h < L ? h : L;
      }
    }
    if (lane == 0 && ibeg == 0) out[0] = 0ull;
    for (int i0 = ibeg; i0 < iend; i0 += 32) {
      const int i = i0 + lane;
      unsigned long long inc = i < iend ? sc[(rev ? L - 1 - i : i) * IW] : 0ull;  // signed: IW == 1
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
      }
      if (i < iend) out[i + 1] = run + inc;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
  }

  // ---- order of E and O 2^N for the - operand (top-down compare)
  int order = 1;
  if (o_neg >= 0) {
    int ord = 0;
    for (int base = m - 1; base >= 0 && ord == 0; base -= 32) {
      const int q = base - lane;
      u32 e = 0u, ov = 0u;
      if (q >= 0) {
        Cur1 ce, co;
        ce.init(q, 0, S);
        co.init(q, N, S);
        e = ce.template bits<IW>(sc, 0, S, b);
        ov = co.template bits<IW>(sc, 1, S, b);
      }
      const unsigned diff = __ballot_sync(0xffffffffu, e != ov);
      if (diff) {
        const int l = __ffs(diff) - 1;  // lowest lane = highest digit
        ord = __shfl_sync(0xffffffffu, e > ov ? 1 : -1, l);
      }
    }
    order = ord >= 0 ? 1 : -1;
  }
  const bool flip = o_neg >= 0 && A.op[o_neg].kind == 3 && (L & 1) == 0;  // pack.py:106-109
  const int negative = (order < 0) != flip ? 1 : 0;

  u32* outp = o_pos >= 0 ? A.op[o_pos].out + (long long)pair * A.op[o_pos].out_pair_stride : nullptr;
  u32* outn = o_neg >= 0 ? A.op[o_neg].out + (long long)pair * A.op[o_neg].out_pair_stride : nullptr;
  int cinp = 0, cinn = 0;  // chunk carry-in (+ stream: 0/1; - stream: 0/-1 stored as 0/1)
  StreamAcc tp{0, 0u}, tn{0, 0u};
  for (int c0 = 0; c0 < m; c0 += W1_CH) {
    const int q0 = c0 + lane * W1_V;
    Cur1 ce, co;
    Str1 se, so;
    if (IW == 1) {
      if (q0 < m) {
        se.init(q0, 0, S, 0, sc);
        so.init(q0, N, S, 1, sc);
      }
    } else {
      ce.init(q0, 0, S);
      co.init(q0, N, S);
    }
    u32 dp[W1_V], dn[W1_V];
    u32 cp = 0u, cn = 0u;  // local carry (+) / borrow (-) with carry-in 0
    u32 allFp = 0xffffffffu, allZn = 0u;
#pragma unroll
    for (int v = 0; v < W1_V; v++) {
      u32 e = 0u, ov = 0u;
      if (IW == 1) {
        if (q0 + v < m) {
          e = se.next(S, sc);
          ov = so.next(S, sc);
        }
      } else {
        if (q0 + v < m) {
          e = ce.template bits<IW>(sc, 0, S, b);
          ov = co.template bits<IW>(sc, 1, S, b);
        }
        ce.next(S);
        co.next(S);
      }
      // + : e + o + carry
      const unsigned long long sp = (unsigned long long)e + ov + cp;
      dp[v] = (u32)sp;
      cp = (u32)(sp >> 32);
      allFp &= dp[v];
      // - : larger - smaller - borrow
      const u32 x = order > 0 ? e : ov, y = order > 0 ? ov : e;
      const unsigned long long sn = (unsigned long long)x - y - cn;
      dn[v] = (u32)sn;
      cn = (u32)(sn >> 63);
      allZn |= dn[v];
    }
    // maps: + carry out for carry-in {0, 1}; - borrow out for borrow-in {0, 1}
    u32 Mp = cp | ((cp | (allFp == 0xffffffffu ? 1u : 0u)) << 1);
    u32 Mn = cn | ((cn | (allZn == 0u ? 1u : 0u)) << 1);
    u32 Ip = Mp, In = Mn;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u32 yp = __shfl_up_sync(0xffffffffu, Ip, d);
      const u32 yn = __shfl_up_sync(0xffffffffu, In, d);
      if (lane >= d) {
        Ip = cmp2(Ip, yp);
        In = cmp2(In, yn);
      }
    }
    const u32 Ep = __shfl_up_sync(0xffffffffu, Ip, 1), En = __shfl_up_sync(0xffffffffu, In, 1);
    const u32 kp = lane ? ((Ep >> cinp) & 1u) : (u32)cinp;
    const u32 kn = lane ? ((En >> cinn) & 1u) : (u32)cinn;
    if (kp) {  // ripple +1
      u32 k = 1u;
#pragma unroll
      for (int v = 0; v < W1_V; v++) {
        dp[v] += k;
        k = (k && dp[v] == 0u) ? 1u : 0u;
      }
    }
    if (kn) {  // ripple -1
      u32 k = 1u;
#pragma unroll
      for (int v = 0; v < W1_V; v++) {
        const u32 old = dn[v];
        dn[v] = old - k;
        k = (k && old == 0u) ? 1u : 0u;
      }
    }
    const u32 totp = __shfl_sync(0xffffffffu, Ip, 31), totn = __shfl_sync(0xffffffffu, In, 31);
    cinp = (int)((totp >> cinp) & 1u);
    cinn = (int)((totn >> cinn) & 1u);
#pragma unroll
    for (int v = 0; v < W1_V; v++) {
      if (q0 + v < m) {
        if (dp[v]) { tp.top = q0 + v + 1; tp.topv = dp[v]; }
        if (dn[v]) { tn.top = q0 + v + 1; tn.topv = dn[v]; }
      }
    }
    if (q0 + W1_V <= m) {
      if (outp) {
        uint4* dst = reinterpret_cast<uint4*>(outp + q0);
        dst[0] = make_uint4(dp[0], dp[1], dp[2], dp[3]);
        dst[1] = make_uint4(dp[4], dp[5], dp[6], dp[7]);
      }
      if (outn) {
        uint4* dst = reinterpret_cast<uint4*>(outn + q0);
        dst[0] = make_uint4(dn[0], dn[1], dn[2], dn[3]);
        dst[1] = make_uint4(dn[4], dn[5], dn[6], dn[7]);
      }
    } else {
#pragma unroll
      for (int v = 0; v < W1_V; v++)
        if (q0 + v < m) {
          if (outp) outp[q0 + v] = dp[v];
          if (outn) outn[q0 + v] = dn[v];
        }
    }
  }
  // the operands fit in m limbs (the plan's +2 bits of margin): no carry out
  if (lane == 0 && ((outp && cinp) || (outn && cinn))) raise_err(A.err, ERR_INEXACT);
  // meta: [sign, bit length] (top nonzero digit: warp max)
  for (int s = 0; s < 2; s++) {
    const int o = s ? o_neg : o_pos;
    if (o < 0) continue;
    const StreamAcc& t = s ? tn : tp;
    const unsigned wmax = __reduce_max_sync(0xffffffffu, (unsigned)t.top);
    u32 v = 0u;
    if (wmax) {
      const int src = __ffs(__ballot_sync(0xffffffffu, (unsigned)t.top == wmax)) - 1;
      v = __shfl_sync(0xffffffffu, t.topv, src);
    }
    if (lane == 0) {
      u32* meta = A.op[o].meta + (long long)pair * A.op[o].meta_pair_stride;
      meta[0] = s ? (u32)negative : 0u;
      meta[1] = wmax ? (u32)(32 * (wmax - 1) + 32 - __clz(v)) : 0u;
    }
  }
}

}  // namespace

// The warp-per-job path applies to one-word coefficients with 2N >= 32 whose
// staged vectors fit: every op shares the vector length and in_words == 1.
bool pack_w1_ok(const PackArgs& a) {
  static const int en = getenv("KMX_PACK_W1") ? atoi(getenv("KMX_PACK_W1")) : 1;
  if (!en || a.in_words < 1 || a.in_words > 2 || 2 * a.N < 32 || a.b > 2 * a.N || a.nops < 1) return false;
  for (int i = 0; i < a.nops; i++)
    if (a.op[i].len != a.op[0].len || a.op[i].prefix_pair_stride < 0) return false;
  const size_t smem = (size_t)W1_WARPS * (a.op[0].len + W1_PAD) * a.in_words * 4;
  return smem <= 200 * 1024;
}

template <int IW>
cudaError_t launch_w1(const PackArgs& a0, int njobs, bool paired, cudaStream_t st) {
  // signed inputs: hand the second half of each polynomial's prefix sums to its reversed job
  // (ks2 / ks4: ops [f: P][g: P], kind 0 carries the prefix pointer, kind 2 is the reversed pack)
  PackArgs a = a0;
  int psplit = 0;
  static const int en_split = getenv("KMX_PACK_PSPLIT") ? atoi(getenv("KMX_PACK_PSPLIT")) : 1;
  if (en_split && a.bias && (a.nops & 1) == 0 && a.op[0].len >= 64) {
    const int half = a.nops / 2;
    int src[2] = {-1, -1}, dst[2] = {-1, -1};
    for (int g = 0; g < 2; g++)
      for (int i = g * half; i < (g + 1) * half; i++) {
        if (a.op[i].prefix && a.op[i].kind == 0) src[g] = i;
        if (!a.op[i].prefix && a.op[i].kind == 2) dst[g] = i;
      }
    if (src[0] >= 0 && dst[0] >= 0 && src[1] >= 0 && dst[1] >= 0) {
      for (int g = 0; g < 2; g++) {
        a.op[dst[g]].prefix = a.op[src[g]].prefix;
        a.op[dst[g]].prefix_pair_stride = a.op[src[g]].prefix_pair_stride;
      }
      psplit = 1;
    }
  }
  // small batches (config 1: 256 jobs): one warp per CTA, spread over more SMs
  const int wpc = njobs < 148 * 2 * W1_WARPS ? 1 : W1_WARPS;
  const size_t smem = (size_t)wpc * (a.op[0].len + W1_PAD) * IW * 4;
  static size_t s_set = 0;
  if (smem > 48 * 1024 && smem > s_set) {
    cudaError_t e = cudaFuncSetAttribute(k_pack_w1<IW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    s_set = smem;
  }
  k_pack_w1<IW><<<(njobs + wpc - 1) / wpc, 32 * wpc, smem, st>>>(a, paired ? 1 : 0, njobs, psplit);
  return cudaGetLastError();
}

cudaError_t launch_pack_w1(const PackArgs& a, int batch, bool paired, cudaStream_t st) {
  const int njobs = batch * (paired ? a.nops / 2 : a.nops);
  if (njobs == 0) return cudaSuccess;
  return a.in_words == 1 ? launch_w1<1>(a, njobs, paired, st) : launch_w1<2>(a, njobs, paired, st);
}

}  // namespace kmx
