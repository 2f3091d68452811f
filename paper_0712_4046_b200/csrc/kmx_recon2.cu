// kmx_recon2.cu -- K4 for digits of at most 64 bits: one CTA per PAIR.
//
// The same recurrence and the same speculate / scan / verify rounds as
// k_recon_par (kmx_ks.cu; ksint.py:137-179): lo[j+1] = lo[j-1] + c_j + e_j
// with c_j = fwd[j+1] - rev[j] and e_j = eps_j - delta_j, every thread owning
// 8 consecutive steps of one stream.  What differs is where the data lives:
//   * a thread's 8 + 9 digits are loaded ONCE from global memory into
//     registers (no shared-memory copy of the streams, no per-step loads in
//     the walks; the c-sums, both walks and the checks run on registers);
//   * both reconstruction streams of a pair (ks4: even and odd coefficients)
//     share the CTA, so the pair's coefficients leave as ONE contiguous
//     record array: the walks drop (lo, hi) pairs into a conflict-free
//     shared-memory transpose, an output pass reads them back in coefficient
//     order, applies the signed correction (prefix sums read coalesced from
//     L2), and the final words go out as aligned 16-byte stores;
//   * scans are warp shuffles plus one small cross-warp table.
// Streams of up to 8 * 1024 / ns steps; longer ones, wider digits and the
// carry-reporting API calls stay on k_recon_par / k_recon.
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

namespace {

constexpr int R2_V = 8;       // steps per thread
constexpr int R2_MAXIT = 8;   // speculation rounds before the sequential fallback
constexpr int R2_MAXT = 1024;

template <int DW>
__device__ __forceinline__ u64 r2_ld(const u32* p, int d) {
  if (DW == 1) return (u64)__ldg(p + d);
  return __ldg(reinterpret_cast<const unsigned long long*>(p) + d);
}

// The signed correction (BiasFix) on a value in registers:
// v - S 2^(b-1) + cnt 2^(2b-2) = v + (cnt 2^(b-1) - S) 2^(b-1); the bracket fits a signed 64-bit word.
__device__ __forceinline__ void r2_bias(u64& lo, u64& hi, u64 S, int cnt, int sh) {
  const i64 D = (i64)(((u64)cnt << sh) - S);
  const u64 dlo = (u64)D << sh;
  const u64 dhi = (u64)(sh ? (D >> (64 - sh)) : (D >> 63));
  const u64 l1 = lo + dlo;
  hi = hi + dhi + (l1 < lo ? 1ull : 0ull);
  lo = l1;
}

// One step of the reference recurrence (ksint.py:153-169) on registers.
#define R2_STEP(FJ1, RJ1)                                        \
  {                                                               \
    const u64 rj1_ = (RJ1), fj1_ = (FJ1);                         \
    const u32 eps_ = lo_cur > rj1_;                               \
    h = (rj - lo_prev - eps_) & m64;                              \
    const u64 nxt_ = (fj1_ - h - fc) & m64;                       \
    const u32 br_ = h + fc > fj1_;                                \
    ej = (int)eps_ - (int)fc;                                     \
    fc = br_;                                                     \
    lo_out = lo_cur;                                              \
    lo_prev = lo_cur;                                             \
    lo_cur = nxt_;                                                \
    rj = rj1_;                                                    \
  }

struct R2State { u64 lo_prev, lo_cur, rj; u32 fc; };

// A thread's (up to) 8 steps from state st; returns the packed e-sums
// n0 + 65536 n1 (by parity of j+1; |sums| < 2^15).  The check hi != 2^W - 1
// (ksint.py:157-158) is made on every coefficient in the output pass.
// FULL: all 8 steps owned (no guards).  STORE: (lo, hi) pairs into the transpose.
template <bool FULL, bool STORE>
__device__ __forceinline__ int r2_walk(R2State& st, const u64 (&fd)[R2_V], const u64 (&rd)[R2_V + 1], int ns_own,
                                       u64 m64, uint4* tslot, int RS) {
  u64 lo_prev = st.lo_prev, lo_cur = st.lo_cur, rj = st.rj;
  u32 fc = st.fc;
  int n = 0;
#pragma unroll
  for (int i = 0; i < R2_V; i++) {
    if (FULL || i < ns_own) {
      u64 h, lo_out;
      int ej;
      R2_STEP(fd[i], rd[i + 1]);
      n += (i & 1) ? ej : ej * 65536;
      if (STORE) tslot[i * RS] = make_uint4((u32)lo_out, (u32)(lo_out >> 32), (u32)h, (u32)(h >> 32));
    }
  }
  st.lo_prev = lo_prev; st.lo_cur = lo_cur; st.rj = rj; st.fc = fc;
  return n;
}

template <int DW>
__global__ void __launch_bounds__(R2_MAXT, 1) k_recon_pair(ReconArgs a, int TS, int aligned, int pf_off) {
  extern __shared__ __align__(16) unsigned char r2s[];
  __shared__ u64 sc_part[R2_MAXT / 32][2];
  __shared__ int se_part[R2_MAXT / 32];
  __shared__ u32 sd_end[R2_MAXT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pair = blockIdx.x;
  const int si = tid >= TS ? 1 : 0, t = tid - (si ? TS : 0);  // stream, thread inside the stream's group
  const int w0 = si ? (TS >> 5) : 0;                          // the group's first warp
  const ReconStream S = si == 0 ? a.s[0] : a.s[1];
  const int W = a.W, count = S.count, nsteps = count - 1;
  const u64 m64 = W >= 64 ? ~0ull : ((1ull << W) - 1ull);
  const u32* F = a.dbuf + ((long long)pair * a.dslots_pair + S.fslot) * a.dslot_stride;
  const u32* R = a.dbuf + ((long long)pair * a.dslots_pair + S.rslot) * a.dslot_stride;
  // signed inputs: the pair's prefix sums (PF | PG) copied into shared memory
  // in the background; the output pass reads them after the walks
  u64* spf = reinterpret_cast<u64*>(r2s + pf_off);
  if (a.bias.enabled) {
    const unsigned long long* PFg = a.bias.pf + (long long)pair * a.bias.pair_stride;
    const int ne = a.bias.lf + a.bias.lg + 2;
    const u32 sdst = (u32)__cvta_generic_to_shared(spf);
    if (((reinterpret_cast<uintptr_t>(PFg) & 15) == 0) && !(ne & 1)) {
      for (int i = tid; i < (ne >> 1); i += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst + 16u * i), "l"(PFg + 2 * i));
    } else {
      for (int i = tid; i < ne; i += blockDim.x)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sdst + 8u * i), "l"(PFg + i));
    }
    asm volatile("cp.async.commit_group;");
  }
  const int s0 = min(t * R2_V, nsteps), s1 = min(s0 + R2_V, nsteps);
  const int ns_own = s1 - s0;                       // steps this thread owns (0..8)
  const bool full = __all_sync(0xffffffffu, ns_own == R2_V);  // warp-uniform: unguarded code

  // ---- digits into registers: fd[i] = fwd[s0+1+i], rd[i] = rev[s0+i] (indices clamped to the
  // stream's count+1 digits; steps past ns_own are never evaluated)
  u64 fd[R2_V], rd[R2_V + 1];
  const bool vec = ((reinterpret_cast<uintptr_t>(F) | reinterpret_cast<uintptr_t>(R)) & 15) == 0;
  if (full && DW == 2 && vec) {
    // s0 = 8t: rev[s0..s0+7] and fwd[s0+2..s0+7] as 16-byte loads (digit pairs)
    const ulonglong2* R2 = reinterpret_cast<const ulonglong2*>(R) + (s0 >> 1);
    const ulonglong2* F2 = reinterpret_cast<const ulonglong2*>(F) + (s0 >> 1);
#pragma unroll
    for (int i = 0; i < R2_V / 2; i++) {
      const ulonglong2 v = __ldg(R2 + i);
      rd[2 * i] = v.x; rd[2 * i + 1] = v.y;
    }
    rd[R2_V] = r2_ld<DW>(R, s0 + R2_V);
    fd[0] = r2_ld<DW>(F, s0 + 1);
#pragma unroll
    for (int i = 1; i < R2_V / 2; i++) {
      const ulonglong2 v = __ldg(F2 + i);
      fd[2 * i - 1] = v.x; fd[2 * i] = v.y;
    }
    fd[R2_V - 1] = r2_ld<DW>(F, s0 + R2_V);
  } else if (full) {
#pragma unroll
    for (int i = 0; i < R2_V; i++) fd[i] = r2_ld<DW>(F, s0 + 1 + i);
#pragma unroll
    for (int i = 0; i <= R2_V; i++) rd[i] = r2_ld<DW>(R, s0 + i);
  } else {
#pragma unroll
    for (int i = 0; i < R2_V; i++) fd[i] = r2_ld<DW>(F, min(s0 + 1 + i, count));
#pragma unroll
    for (int i = 0; i <= R2_V; i++) rd[i] = r2_ld<DW>(R, min(s0 + i, count));
  }
  const u64 f0 = r2_ld<DW>(F, 0);

  // ---- exact chain bases: exclusive scan of the c-sums by parity of j+1
  // (s0 is even, so local step i has (j+1) odd exactly when i is even)
  u64 cs0 = 0, cs1 = 0;
#pragma unroll
  for (int i = 0; i < R2_V; i++) {
    const u64 c = (full || i < ns_own) ? fd[i] - rd[i] : 0ull;
    if (i & 1) cs0 += c; else cs1 += c;
  }
  {
    u64 i0 = cs0, i1 = cs1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 p0 = __shfl_up_sync(0xffffffffu, i0, o), p1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) { i0 += p0; i1 += p1; }
    }
    if (lane == 31) { sc_part[warp][0] = i0; sc_part[warp][1] = i1; }
    __syncthreads();
    u64 q0 = 0, q1 = 0;
    for (int w = w0; w < warp; w++) { q0 += sc_part[w][0]; q1 += sc_part[w][1]; }
    cs0 = q0 + i0 - cs0;
    cs1 = q1 + i1 - cs1;
  }
  cs0 = (cs0 + f0) & m64;  // even chain starts at lo[0] = fwd[0], odd at lo[-1] = 0
  cs1 &= m64;

  // transpose buffer: (lo, hi) of coefficient j = 8t + i of stream si at 16-byte slot
  // si * (8 RS + 4) + i * RS + t, RS = TS + 1
  uint4* tb = reinterpret_cast<uint4*>(r2s);
  const int RS = TS + 1;
  const int sbase = si ? 8 * RS + 4 : 0;
  uint4* tslot = tb + sbase + t;

  int E = 0;  // packed corrections at the segment start: E0 + 65536 E1
  u32 dstart = 0;
  bool converged = false, bfin = false;
  int nprev = 0;    // this thread's own e-sums and end delta in the previous round
  u32 fcprev = 0;
  const bool owner = t == (nsteps > 0 ? (nsteps - 1) / R2_V : 0);  // holds the state after the last step
  R2State st;
  for (int it = 0; it < R2_MAXIT; it++) {
    const int E0 = (int)(short)(E & 0xffff), E1 = (E - E0) >> 16;
    st.lo_cur = (cs0 + (u64)(i64)E0) & m64;
    st.lo_prev = s0 == 0 ? 0ull : ((cs1 + (u64)(i64)E1) & m64);
    st.rj = rd[0];
    st.fc = dstart;
    // rounds after the first store: the round that converges started from the exact state
    int n;
    if (full) n = it ? r2_walk<true, true>(st, fd, rd, ns_own, m64, tslot, RS)
                     : r2_walk<true, false>(st, fd, rd, ns_own, m64, tslot, RS);
    else n = it ? r2_walk<false, true>(st, fd, rd, ns_own, m64, tslot, RS)
                : r2_walk<false, false>(st, fd, rd, ns_own, m64, tslot, RS);
    if (it > 0) {
      if (owner) {
        // last coefficient and the consistency checks (ksint.py:170-177), kept if this round converges
        if (nsteps == 0) { st.lo_prev = 0; st.lo_cur = f0; st.fc = 0; }
        const u64 h = (st.rj - (count >= 2 ? st.lo_prev : 0ull)) & m64;
        const u64 rlast = r2_ld<DW>(R, count), flast = r2_ld<DW>(F, count);
        bfin = st.lo_cur != rlast || (h + st.fc > flast) || (flast - h - st.fc) != 0ull;
        const int j = count - 1;
        tb[sbase + (j & 7) * RS + (j >> 3)] = make_uint4((u32)st.lo_cur, (u32)(st.lo_cur >> 32), (u32)h, (u32)(h >> 32));
      }
      // Fixed point: every thread reproduced its own e-sums and end delta, so the scans -- and
      // with them every start state of this round -- are what this round itself implies.
      asm volatile("cp.async.wait_group 0;");
      converged = __syncthreads_and(n == nprev && st.fc == fcprev);
      if (converged) break;
    }
    nprev = n; fcprev = st.fc;
    // exclusive scan of the e-sums over the stream's group; delta handed to the next thread
    int x = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int p = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += p;
    }
    u32 dnew = __shfl_up_sync(0xffffffffu, st.fc, 1);
    if (lane == 31) { se_part[warp] = x; sd_end[warp] = st.fc; }
    __syncthreads();
    int q = 0;
    for (int w = w0; w < warp; w++) q += se_part[w];
    if (lane == 0) dnew = warp > w0 ? sd_end[warp - 1] : 0u;
    E = q + x - n;
    dstart = dnew;
  }

  bool raise = false;
  if (converged) {
    raise = bfin;
  } else {
    if (t == 0) {
      // sequential fallback: one thread per stream walks it from the exact start
      if (a.diag) atomicAdd(a.diag, 1u);
      u64 lo_prev = 0, lo_cur = f0, rj = r2_ld<DW>(R, 0);
      u32 fc = 0;
      for (int j = 0; j < nsteps; j++) {
        u64 h, lo_out;
        int ej;
        R2_STEP(r2_ld<DW>(F, j + 1), r2_ld<DW>(R, j + 1));
        (void)ej;
        tb[sbase + (j & 7) * RS + (j >> 3)] = make_uint4((u32)lo_out, (u32)(lo_out >> 32), (u32)h, (u32)(h >> 32));
      }
      const u64 h = (rj - (count >= 2 ? lo_prev : 0ull)) & m64;
      bool b2 = false;
      const u64 rlast = r2_ld<DW>(R, count), flast = r2_ld<DW>(F, count);
      b2 |= lo_cur != rlast;
      b2 |= (h + fc > flast) || (flast - h - fc) != 0ull;
      raise = b2;
      const int j = count - 1;
      tb[sbase + (j & 7) * RS + (j >> 3)] = make_uint4((u32)lo_cur, (u32)(lo_cur >> 32), (u32)h, (u32)(h >> 32));
    }
    __syncthreads();
  }
  // ---- output pass: coefficient k = tid + T r, in coefficient order (indices clamped to the
  // last coefficient so that the loads of all rounds can be in flight together)
  const int T = blockDim.x, ow = a.out_words;
  const int klen = a.ns == 1 ? a.s[0].count : a.s[0].count + a.s[1].count;
  const bool two = a.ns == 2;
  const int sb1 = 8 * RS + 4;
  u64 olo[R2_V], ohi[R2_V];
  if (a.bias.enabled) {
    const int lf = a.bias.lf, lg = a.bias.lg, sh = a.bias.b - 1;
    const u64* PF = spf;
    const u64* PG = spf + lf + 1;
#pragma unroll
    for (int r = 0; r < R2_V; r++) {
      const int k = min(tid + T * r, klen - 1);
      const int j = two ? k >> 1 : k;
      const uint4 v = tb[((two && (k & 1)) ? sb1 : 0) + (j & 7) * RS + (j >> 3)];
      const u64 lo = (u64)v.x | ((u64)v.y << 32), hi = (u64)v.z | ((u64)v.w << 32);
      raise |= hi == m64;
      u64 v0, v1;
      if (W >= 64) { v0 = lo; v1 = hi; }
      else { v0 = lo | (hi << W); v1 = hi >> (64 - W); }
      const int i1 = min(k, lf - 1), i0 = max(k - lg + 1, 0);
      const u64 S = (PF[i1 + 1] - PF[i0]) + (PG[min(k, lg - 1) + 1] - PG[max(k - lf + 1, 0)]);
      r2_bias(v0, v1, S, i1 - i0 + 1, sh);
      olo[r] = v0; ohi[r] = v1;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R2_V; r++) {
      const int k = min(tid + T * r, klen - 1);
      const int j = two ? k >> 1 : k;
      const uint4 v = tb[((two && (k & 1)) ? sb1 : 0) + (j & 7) * RS + (j >> 3)];
      const u64 lo = (u64)v.x | ((u64)v.y << 32), hi = (u64)v.z | ((u64)v.w << 32);
      raise |= hi == m64;
      if (W >= 64) { olo[r] = lo; ohi[r] = hi; }
      else { olo[r] = lo | (hi << W); ohi[r] = hi >> (64 - W); }
    }
  }
  if (raise) raise_err(a.err, ERR_RECON);
  __syncthreads();
  // final words into shared memory at the global address's phase, then 16-byte stores
  u32* H = a.h + (long long)pair * a.h_pair_stride;
  const int ph = aligned ? (int)((reinterpret_cast<uintptr_t>(H) >> 2) & 3) : 0;
  u32* fw = reinterpret_cast<u32*>(r2s);
  if (ow == 3) {
#pragma unroll
    for (int r = 0; r < R2_V; r++) {
      const int k = tid + T * r;
      if (k < klen) {
        u32* d = fw + ph + 3 * k;
        d[0] = (u32)olo[r]; d[1] = (u32)(olo[r] >> 32); d[2] = (u32)ohi[r];
      }
    }
  } else {
#pragma unroll
    for (int r = 0; r < R2_V; r++) {
      const int k = tid + T * r;
      if (k < klen) {
        u32* d = fw + ph + (size_t)k * ow;
        const u32 ext = (a.bias.enabled && (ohi[r] >> 63)) ? 0xffffffffu : 0u;
        d[0] = (u32)olo[r];
        if (ow > 1) d[1] = (u32)(olo[r] >> 32);
        if (ow > 2) d[2] = (u32)ohi[r];
        if (ow > 3) d[3] = (u32)(ohi[r] >> 32);
        for (int w = 4; w < ow; w++) d[w] = ext;
      }
    }
  }
  __syncthreads();
  const int nw = klen * ow;
  if (aligned) {
    u32* Hb = H - ph;  // 16-byte aligned
    const int qa = (ph + 3) >> 2, qb = (ph + nw) >> 2;  // 16-byte chunks [qa, qb) lie inside the pair's words
    for (int q = qa + tid; q < qb; q += T)
      *reinterpret_cast<uint4*>(Hb + 4 * q) = *reinterpret_cast<const uint4*>(fw + 4 * q);
    if (tid < 8) {  // the words before the first and after the last whole chunk
      const int hend = qb >= qa ? 4 * qa : ph + nw, tbeg = qb >= qa ? 4 * qb : ph + nw;
      const int w = tid < 4 ? ph + tid : tbeg + tid - 4;
      if (tid < 4 ? w < hend : w < ph + nw) Hb[w] = fw[w];
    }
  } else {
    for (int w = tid; w < nw; w += T) H[w] = fw[w];
  }
}

}  // namespace

// ------------------------------------------------------------------------
// Signed correction as a streaming pass (ks1 / ks3, whose finish writes the
// coefficients itself): h[k] = h'[k] - S_k 2^(b-1) + cnt_k 2^(2b-2) in place,
// one thread per coefficient, the prefix sums and the records read coalesced.
// Inside the finish the same correction costs four dependent L2 loads per
// coefficient in the latency-critical chunk loop (c2 ks1 / ks3 finish 62 us
// against 31-36 us for unsigned inputs of the same shape).
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bias_apply(BiasFix bf, u32* h, int ow, int klen, long long h_pair_stride) {
  const int pair = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= klen) return;
  const unsigned long long* PF = bf.pf + (long long)pair * bf.pair_stride;
  const int lf = bf.lf, lg = bf.lg;
  const unsigned long long* PG = PF + lf + 1;
  const int i1 = min(k, lf - 1), i0 = max(k - lg + 1, 0);
  const u64 S = (__ldg(PF + i1 + 1) - __ldg(PF + i0)) + (__ldg(PG + min(k, lg - 1) + 1) - __ldg(PG + max(k - lf + 1, 0)));
  u32* hk = h + (long long)pair * h_pair_stride + (long long)k * ow;
  u64 lo = hk[0], hi = 0;
  if (ow > 1) lo |= (u64)hk[1] << 32;
  if (ow > 2) hi = hk[2];
  if (ow > 3) hi |= (u64)hk[3] << 32;
  r2_bias(lo, hi, S, i1 - i0 + 1, bf.b - 1);
  hk[0] = (u32)lo;
  if (ow > 1) hk[1] = (u32)(lo >> 32);
  if (ow > 2) hk[2] = (u32)hi;
  if (ow > 3) hk[3] = (u32)(hi >> 32);
  const u32 ext = (hi >> 63) ? 0xffffffffu : 0u;
  for (int w = 4; w < ow; w++) hk[w] = ext;
}

// Launch geometry: threads per stream and the shared-memory layout (transpose slots / final
// words, whichever is larger, then the signed path's prefix sums).
struct R2Geom { int TS, T, pf_off; size_t smem; };
static R2Geom r2_geometry(const ReconArgs& a) {
  int maxcount = a.s[0].count;
  if (a.ns == 2 && a.s[1].count > maxcount) maxcount = a.s[1].count;
  R2Geom g;
  // 8 TS >= count: the group's threads cover the steps, and 8 T the pair's coefficients
  g.TS = ((maxcount + R2_V - 1) / R2_V + 31) & ~31;
  g.T = g.TS * a.ns;
  const int klen = a.ns == 1 ? a.s[0].count : a.s[0].count + a.s[1].count;
  const size_t tbytes = (size_t)(a.ns * (8 * (g.TS + 1) + 4)) * 16;
  const size_t fbytes = ((size_t)klen * a.out_words + 8) * 4;
  g.smem = ((tbytes > fbytes ? tbytes : fbytes) + 15) & ~(size_t)15;
  g.pf_off = (int)g.smem;
  if (a.bias.enabled) g.smem += ((size_t)(a.bias.lf + a.bias.lg + 2) * 8 + 15) & ~(size_t)15;
  return g;
}

// One CTA per pair: digits of at most two words, no carry report, streams
// short enough for 8 steps per thread.  KMX_RECON_PAIR=0 disables, 2 forces it for short streams too.
bool recon_pair_ok(const ReconArgs& a) {
  static const int en = getenv("KMX_RECON_PAIR") ? atoi(getenv("KMX_RECON_PAIR")) : 1;
  if (!en || a.carries || a.sequential || a.dwords > 2 || a.ns < 1 || a.ns > 2 || a.batch < 1) return false;
  if (a.dwords == 2 && ((reinterpret_cast<uintptr_t>(a.dbuf) & 7) || (a.dslot_stride & 1))) return false;
  int maxcount = a.s[0].count;
  if (a.ns == 2) {
    // interleaved even / odd coefficients (ks4): stream 0 at 0, 2, ..., stream 1 at 1, 3, ...
    if (a.s[0].pos0 != 0 || a.s[1].pos0 != 1 || a.s[0].pstride != 2 || a.s[1].pstride != 2) return false;
    if (a.s[1].count != a.s[0].count && a.s[1].count != a.s[0].count - 1) return false;
    if (a.s[1].count < 1) return false;
    if (a.s[1].count > maxcount) maxcount = a.s[1].count;
  } else if (a.s[0].pos0 != 0 || a.s[0].pstride != 1) {
    return false;
  }
  if (a.s[0].count < 1) return false;
  // measured over config 5 (KMX_RECON_PAIR=2 forces): streams of fewer than 256 digits leave the
  // pair's CTA at one or two warps and k_recon_par is 8-10% faster there
  if (en != 2 && maxcount < 256) return false;
  const R2Geom g = r2_geometry(a);
  return g.T <= R2_MAXT && g.smem <= 200 * 1024;  // (a caller's wide out_words can outgrow the final-word buffer)
}

cudaError_t launch_recon_pair(const ReconArgs& a, cudaStream_t st) {
  const R2Geom g = r2_geometry(a);
  if (g.T > R2_MAXT || g.smem > 200 * 1024) return cudaErrorInvalidValue;
  const int aligned = (reinterpret_cast<uintptr_t>(a.h) & 3) == 0 ? 1 : 0;
  auto kern = a.dwords == 1 ? k_recon_pair<1> : k_recon_pair<2>;
  if (g.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<a.batch, g.T, g.smem, st>>>(a, g.TS, aligned, g.pf_off);
  return cudaGetLastError();
}

// In-place signed correction of [batch][klen][ow] coefficient records (values below 2^128).
cudaError_t launch_bias_apply(const BiasFix& bf, uint32_t* h, int out_words, int klen, long long h_pair_stride, int batch,
                              cudaStream_t st) {
  if (batch < 1 || klen < 1) return cudaSuccess;
  if (batch > 65535) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((klen + 255) / 256), (unsigned)batch);
  k_bias_apply<<<grid, 256, 0, st>>>(bf, h, out_words, klen, h_pair_stride);
  return cudaGetLastError();
}

}  // namespace kmx
