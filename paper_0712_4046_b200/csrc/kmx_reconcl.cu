// kmx_reconcl.cu -- K4 for FEW, LONG streams: one thread-block CLUSTER per
// reconstruction stream (ksint.py:137-179).
//
// k_recon_par (kmx_ks.cu) gives a stream one CTA.  At the BASELINE config 4
// (32 pairs, 4097- and 8191-digit streams of 134 bits) that is 32 or 64 CTAs on
// 148 SMs, each walking thousands of steps, and the 8191-digit streams do not
// fit one CTA's shared memory, so their walks read global memory step by step.
// Here C = 2..8 CTAs of a cluster share a stream: CTA r stages and owns the
// steps [r spc, (r+1) spc), and the three things the segments exchange --
// the exact chain bases (prefix of the c-sums), the corrections (prefix of the
// e-sums with the delta handed to the next thread) and the convergence vote --
// cross the CTA boundary through distributed shared memory with one cluster
// barrier each.  The recurrence, the speculate / verify rounds and the checks
// are those of k_recon_par: lo[j+1] = lo[j-1] + c_j + e_j, c_j = fwd[j+1] -
// rev[j], e_j = eps_j - delta_j; a round whose threads all reproduce their own
// e-sums and end delta started from the exact state, and its stores are the
// output.  Unsigned coefficients only (signed inputs have digits of at most
// 64 bits and take the pair kernel, kmx_recon2.cu).
#include <cooperative_groups.h>
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace cg = cooperative_groups;

namespace kmx {

namespace {

constexpr int RC_MAXT = 512;
constexpr int RC_MAXIT = 8;
constexpr int RC_MAXW = RC_MAXT / 32;

template <int NW>
struct QW { u32 w[NW]; };

template <int NW>
__device__ __forceinline__ void q_ld(QW<NW>& x, const u32* p) {
#pragma unroll
  for (int i = 0; i < NW; i++) x.w[i] = p[i];
}
template <int NW>
__device__ __forceinline__ void q_zero(QW<NW>& x) {
#pragma unroll
  for (int i = 0; i < NW; i++) x.w[i] = 0u;
}
// r = x - y - bin (mod 2^(32 NW)); returns the borrow out
template <int NW>
__device__ __forceinline__ u32 q_sub(QW<NW>& r, const QW<NW>& x, const QW<NW>& y, u32 bin) {
  u32 br = bin;
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const u64 t = (u64)x.w[i] - y.w[i] - br;
    r.w[i] = (u32)t;
    br = (u32)(t >> 63);
  }
  return br;
}
template <int NW>
__device__ __forceinline__ void q_add(QW<NW>& r, const QW<NW>& x, const QW<NW>& y) {
  u32 c = 0;
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const u64 t = (u64)x.w[i] + y.w[i] + c;
    r.w[i] = (u32)t;
    c = (u32)(t >> 32);
  }
}
template <int NW>
__device__ __forceinline__ void q_add_small(QW<NW>& r, const QW<NW>& x, int e) {  // r = x + e (sign-extended)
  const u32 ext = e < 0 ? 0xffffffffu : 0u;
  u32 c = 0;
#pragma unroll
  for (int i = 0; i < NW; i++) {
    const u64 t = (u64)x.w[i] + (i == 0 ? (u32)e : ext) + c;
    r.w[i] = (u32)t;
    c = (u32)(t >> 32);
  }
}
template <int NW>
__device__ __forceinline__ bool q_gt(const QW<NW>& x, const QW<NW>& y) {  // x > y
  QW<NW> t;
  return q_sub(t, y, x, 0u) != 0u;
}
template <int NW>
__device__ __forceinline__ bool q_eq(const QW<NW>& x, const QW<NW>& y) {
  bool e = true;
#pragma unroll
  for (int i = 0; i < NW; i++) e &= x.w[i] == y.w[i];
  return e;
}
template <int NW>
__device__ __forceinline__ bool q_is_zero(const QW<NW>& x) {
  u32 o = 0u;
#pragma unroll
  for (int i = 0; i < NW; i++) o |= x.w[i];
  return o == 0u;
}
// coefficient lo + hi 2^W (lo < 2^W) into ow words
template <int NW>
__device__ __forceinline__ void q_store(u32* dst, int ow, const QW<NW>& lo, const QW<NW>& hi, int W) {
  const int ws = W >> 5, bs = W & 31;
#pragma unroll
  for (int w = 0; w < 2 * NW + 1; w++) {
    if (w < ow) {
      u32 x = w < NW ? lo.w[w] : 0u;
#pragma unroll
      for (int k = 0; k < NW; k++) {
        if (w == ws + k) x |= hi.w[k] << bs;
        if (bs && w == ws + k + 1) x |= hi.w[k] >> (32 - bs);
      }
      dst[w] = x;
    }
  }
  for (int w = 2 * NW + 1; w < ow; w++) dst[w] = 0u;
}

template <int NW>
struct RcShared {
  u32 ctot[2 * NW];             // this CTA's c-sum totals (even chain, odd chain)
  int etot[2][4];               // by round parity: e-sum totals (even, odd), the last thread's end delta
  int ok[2];                    // by round parity: every thread of this CTA reproduced its sums
  u32 wq[2 * NW * RC_MAXW];     // block scans: per-warp partials
  int wi[2 * RC_MAXW];
  unsigned char dend[RC_MAXT];
};

// Block-wide exclusive scan of a pair of multiword values (mod 2^(32 NW)); tot0 / tot1: the block totals.
template <int NW>
__device__ __forceinline__ void rc_scan_q2(QW<NW>& x0, QW<NW>& x1, QW<NW>& tot0, QW<NW>& tot1, u32* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  QW<NW> i0 = x0, i1 = x1;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    QW<NW> o0, o1;
#pragma unroll
    for (int k = 0; k < NW; k++) {
      o0.w[k] = __shfl_up_sync(0xffffffffu, i0.w[k], off);
      o1.w[k] = __shfl_up_sync(0xffffffffu, i1.w[k], off);
    }
    if (lane >= off) { q_add(i0, i0, o0); q_add(i1, i1, o1); }
  }
  if (lane == 31) {
#pragma unroll
    for (int k = 0; k < NW; k++) { sm[(2 * warp) * NW + k] = i0.w[k]; sm[(2 * warp + 1) * NW + k] = i1.w[k]; }
  }
  __syncthreads();
  QW<NW> p0, p1;
  q_zero(p0); q_zero(p1);
  q_zero(tot0); q_zero(tot1);
  for (int w = 0; w < nw; w++) {
    QW<NW> t0, t1;
    q_ld(t0, sm + (2 * w) * NW);
    q_ld(t1, sm + (2 * w + 1) * NW);
    if (w < warp) { q_add(p0, p0, t0); q_add(p1, p1, t1); }
    q_add(tot0, tot0, t0);
    q_add(tot1, tot1, t1);
  }
  QW<NW> e0, e1;
#pragma unroll
  for (int k = 0; k < NW; k++) {
    e0.w[k] = __shfl_up_sync(0xffffffffu, i0.w[k], 1);
    e1.w[k] = __shfl_up_sync(0xffffffffu, i1.w[k], 1);
  }
  if (lane == 0) { q_zero(e0); q_zero(e1); }
  q_add(x0, p0, e0);
  q_add(x1, p1, e1);
  __syncthreads();
}

// Block-wide exclusive scan of two ints; t0 / t1: the block totals.
__device__ __forceinline__ void rc_scan_i2(int& x0, int& x1, int& t0, int& t1, int* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int i0 = x0, i1 = x1;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o0 = __shfl_up_sync(0xffffffffu, i0, off), o1 = __shfl_up_sync(0xffffffffu, i1, off);
    if (lane >= off) { i0 += o0; i1 += o1; }
  }
  if (lane == 31) { sm[2 * warp] = i0; sm[2 * warp + 1] = i1; }
  __syncthreads();
  int p0 = 0, p1 = 0;
  t0 = 0; t1 = 0;
  for (int w = 0; w < nw; w++) {
    const int a0 = sm[2 * w], a1 = sm[2 * w + 1];
    if (w < warp) { p0 += a0; p1 += a1; }
    t0 += a0; t1 += a1;
  }
  x0 = p0 + i0 - x0;
  x1 = p1 + i1 - x1;
  __syncthreads();
}

template <int NW>
struct RcState {
  QW<NW> lo_prev, lo_cur, rj;  // lo[j-1], lo[j], rev[j]
  u32 fc;                      // delta_j
};

// Steps [j0, j1) of the reference recurrence (ksint.py:153-169).  F / R are indexed by
// (j - jbase) through pos(): staged copies (pad word per 2^lgV digits) or global memory (lgV < 0).
template <int NW, bool STORE>
__device__ __forceinline__ void rc_walk(RcState<NW>& st, int j0, int j1, const u32* F, const u32* R, int jbase, int dw,
                                        int lgV, u32* H, int pos0, int pstride, int ow, int W, u32 topmask,
                                        const QW<NW>& mask, int& e0, int& e1, bool& bad) {
  for (int j = j0; j < j1; j++) {
    const int d = j + 1 - jbase;
    const int pj = d * dw + (lgV >= 0 ? (d >> lgV) : 0);
    QW<NW> rj1, fj1, h, nxt;
    q_ld(rj1, R + pj);
    q_ld(fj1, F + pj);
    const u32 eps = q_gt(st.lo_cur, rj1) ? 1u : 0u;  // ksint.py:154 (strict)
    q_sub(h, st.rj, st.lo_prev, eps);
    h.w[NW - 1] &= topmask;
    bad |= q_eq(h, mask);                            // ksint.py:157-158
    const u32 br = q_sub(nxt, fj1, h, st.fc);        // borrow <=> hi + delta > fwd[j+1]
    nxt.w[NW - 1] &= topmask;
    if (STORE) q_store(H + (long long)(pos0 + (long long)j * pstride) * ow, ow, st.lo_cur, h, W);
    const int ej = (int)eps - (int)st.fc;
    if ((j + 1) & 1) e1 += ej; else e0 += ej;
    st.fc = br;
    st.lo_prev = st.lo_cur;
    st.lo_cur = nxt;
    st.rj = rj1;
  }
}

// last coefficient and the consistency checks (ksint.py:170-177); st: the state after the last step
template <int NW>
__device__ __forceinline__ bool rc_final(const RcState<NW>& st, int count, const QW<NW>& flast, const QW<NW>& rlast,
                                         u32* H, int pos0, int pstride, int ow, int W, u32 topmask,
                                         const QW<NW>& mask) {
  QW<NW> zero, h, hs;
  q_zero(zero);
  q_sub(h, st.rj, count >= 2 ? st.lo_prev : zero, 0u);
  h.w[NW - 1] &= topmask;
  bool b2 = q_eq(h, mask);
  b2 |= !q_eq(st.lo_cur, rlast);
  const u32 br = q_sub(hs, flast, h, st.fc);  // hi + delta == fwd[count]
  b2 |= (br != 0u) || !q_is_zero(hs);
  q_store(H + (long long)(pos0 + (long long)(count - 1) * pstride) * ow, ow, st.lo_cur, h, W);
  return b2;
}

template <int NW>
__global__ void __launch_bounds__(RC_MAXT) k_recon_cl(ReconArgs a, int lgV, int spc) {
  extern __shared__ u32 rcs[];
  __shared__ RcShared<NW> sh;
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.dim_blocks().x, rank = (int)cl.block_rank();
  const int sid = blockIdx.x / C;
  const int pair = sid / a.ns, si = sid - pair * a.ns;
  const ReconStream S = si == 0 ? a.s[0] : a.s[1];
  const int W = a.W, dw = a.dwords, ow = a.out_words, count = S.count, nsteps = count - 1;
  const int tid = threadIdx.x, T = blockDim.x, V = 1 << lgV;
  const u32* Fg = a.dbuf + ((long long)pair * a.dslots_pair + S.fslot) * a.dslot_stride;
  const u32* Rg = a.dbuf + ((long long)pair * a.dslots_pair + S.rslot) * a.dslot_stride;
  u32* H = a.h + (long long)pair * a.h_pair_stride;
  const int topbits = W - 32 * (NW - 1);
  const u32 topmask = topbits >= 32 ? 0xffffffffu : ((1u << topbits) - 1u);
  QW<NW> mask, zero;
#pragma unroll
  for (int i = 0; i < NW; i++) { mask.w[i] = 0xffffffffu; zero.w[i] = 0u; }
  mask.w[NW - 1] &= topmask;

  // this CTA's steps [S0, S1) and its staged digits S0 .. S1 + 1 (<= count) of both streams
  const int S0 = min(rank * spc, nsteps), S1 = min(S0 + spc, nsteps);
  const int nd = S1 - S0 + 2;
  const int slot = nd * dw + (nd >> lgV) + 1;
  u32* Fs = rcs;
  u32* Rs = rcs + slot;
  for (int d = tid; d < nd; d += T) {
    const int pd = d * dw + (d >> lgV);
    const long long g = (long long)(S0 + d) * dw;
    for (int w = 0; w < dw; w++) {
      const unsigned sf = (unsigned)__cvta_generic_to_shared(Fs + pd + w);
      const unsigned sr = (unsigned)__cvta_generic_to_shared(Rs + pd + w);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sf), "l"(Fg + g + w));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sr), "l"(Rg + g + w));
    }
  }
  asm volatile("cp.async.commit_group;");
  asm volatile("cp.async.wait_group 0;");
  __syncthreads();

  const int s0 = min(S0 + tid * V, S1), s1 = min(s0 + V, S1);
  // exact chain bases at the segment start: init + sum of c_j over j < s0, by parity of j + 1
  QW<NW> cs0 = zero, cs1 = zero;
  for (int j = s0; j < s1; j++) {
    const int d1 = j + 1 - S0, d0 = j - S0;
    QW<NW> f1, r0, c;
    q_ld(f1, Fs + d1 * dw + (d1 >> lgV));
    q_ld(r0, Rs + d0 * dw + (d0 >> lgV));
    q_sub(c, f1, r0, 0u);
    if ((j + 1) & 1) q_add(cs1, cs1, c); else q_add(cs0, cs0, c);
  }
  {
    QW<NW> t0, t1;
    rc_scan_q2(cs0, cs1, t0, t1, sh.wq);
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < NW; k++) { sh.ctot[k] = t0.w[k]; sh.ctot[NW + k] = t1.w[k]; }
    }
  }
  cl.sync();
  for (int r = 0; r < rank; r++) {
    const RcShared<NW>* rs = cl.map_shared_rank(&sh, r);
    QW<NW> t0, t1;
    q_ld(t0, rs->ctot);
    q_ld(t1, rs->ctot + NW);
    q_add(cs0, cs0, t0);
    q_add(cs1, cs1, t1);
  }
  {
    QW<NW> f0;
#pragma unroll
    for (int k = 0; k < NW; k++) f0.w[k] = __ldg(Fg + k);
    q_add(cs0, cs0, f0);  // even chain starts at lo[0] = fwd[0], odd at lo[-1] = 0
  }
  cs0.w[NW - 1] &= topmask;
  cs1.w[NW - 1] &= topmask;

  int E0 = 0, E1 = 0;
  u32 dstart = 0;
  int np0 = 0, np1 = 0;
  u32 fcprev = 0;
  bool converged = false, bad = false, bfin = false;
  const bool owner = nsteps > 0 ? (s0 <= nsteps - 1 && nsteps - 1 < s1) : (rank == 0 && tid == 0);
  RcState<NW> st;
  // chain bases of lo[s0] and lo[s0 - 1] (element-wise selects keep them in registers)
  const int p = s0 & 1;
  QW<NW> bcur, bprev;
#pragma unroll
  for (int k = 0; k < NW; k++) { bcur.w[k] = p ? cs1.w[k] : cs0.w[k]; bprev.w[k] = p ? cs0.w[k] : cs1.w[k]; }
  for (int it = 0; it < RC_MAXIT; it++) {
    q_add_small(st.lo_cur, bcur, p ? E1 : E0);
    st.lo_cur.w[NW - 1] &= topmask;
    if (s0 == 0) {
      st.lo_prev = zero;
    } else {
      q_add_small(st.lo_prev, bprev, p ? E0 : E1);
      st.lo_prev.w[NW - 1] &= topmask;
    }
    {
      const int d = s0 - S0;
      q_ld(st.rj, Rs + d * dw + (d >> lgV));
    }
    st.fc = dstart;
    bad = false;
    int n0 = 0, n1 = 0;
    // rounds after the first store: the round that converges started from the exact state
    if (it) rc_walk<NW, true>(st, s0, s1, Fs, Rs, S0, dw, lgV, H, S.pos0, S.pstride, ow, W, topmask, mask, n0, n1, bad);
    else rc_walk<NW, false>(st, s0, s1, Fs, Rs, S0, dw, lgV, H, S.pos0, S.pstride, ow, W, topmask, mask, n0, n1, bad);
    if (it > 0) {
      if (owner) {
        RcState<NW> sf = st;
        if (nsteps == 0) { sf.lo_prev = zero; sf.fc = 0u; }  // lo_cur = fwd[0], rj = rev[0] already
        const int dl = count - S0;
        QW<NW> flast, rlast;
        q_ld(flast, Fs + dl * dw + (dl >> lgV));
        q_ld(rlast, Rs + dl * dw + (dl >> lgV));
        bfin = rc_final(sf, count, flast, rlast, H, S.pos0, S.pstride, ow, W, topmask, mask);
      }
      // Fixed point: every thread of the cluster reproduced its own e-sums and end delta, so the
      // scans -- and with them every start state of this round -- are what the round itself implies.
      const int okb = __syncthreads_and(n0 == np0 && n1 == np1 && st.fc == fcprev);
      if (tid == 0) sh.ok[it & 1] = okb;
      cl.sync();
      bool all = true;
      for (int r = 0; r < C; r++) all &= cl.map_shared_rank(&sh, r)->ok[it & 1] != 0;
      converged = all;
      if (converged) break;
    }
    np0 = n0; np1 = n1; fcprev = st.fc;
    // corrections at the segment starts: exclusive scan of the e-sums over the cluster, delta from
    // the preceding thread
    int t0, t1;
    sh.dend[tid] = (unsigned char)st.fc;
    rc_scan_i2(n0, n1, t0, t1, sh.wi);  // (its barriers order dend)
    if (tid == T - 1) { sh.etot[it & 1][0] = t0; sh.etot[it & 1][1] = t1; sh.etot[it & 1][2] = (int)st.fc; }
    u32 dnew = tid ? (u32)sh.dend[tid - 1] : 0u;
    cl.sync();
    for (int r = 0; r < rank; r++) {
      const RcShared<NW>* rs = cl.map_shared_rank(&sh, r);
      n0 += rs->etot[it & 1][0];
      n1 += rs->etot[it & 1][1];
    }
    if (tid == 0 && rank > 0) dnew = (u32)cl.map_shared_rank(&sh, rank - 1)->etot[it & 1][2];
    E0 = n0; E1 = n1; dstart = dnew;
  }

  bool raise = false;
  if (converged) {
    raise = bad || bfin;
  } else if (rank == 0 && tid == 0) {
    // sequential fallback: one thread walks the whole stream from the exact start (global memory)
    if (a.diag) atomicAdd(a.diag, 1u);
    RcState<NW> sq;
    sq.lo_prev = zero;
#pragma unroll
    for (int k = 0; k < NW; k++) { sq.lo_cur.w[k] = Fg[k]; sq.rj.w[k] = Rg[k]; }
    sq.fc = 0u;
    int q0 = 0, q1 = 0;
    bool b1 = false;
    rc_walk<NW, true>(sq, 0, nsteps, Fg, Rg, 0, dw, -1, H, S.pos0, S.pstride, ow, W, topmask, mask, q0, q1, b1);
    QW<NW> flast, rlast;
#pragma unroll
    for (int k = 0; k < NW; k++) { flast.w[k] = Fg[(long long)count * dw + k]; rlast.w[k] = Rg[(long long)count * dw + k]; }
    raise = rc_final(sq, count, flast, rlast, H, S.pos0, S.pstride, ow, W, topmask, mask) || b1;
  }
  if (raise) raise_err(a.err, ERR_RECON);
  cl.sync();  // no CTA leaves while its shared memory may still be read by its cluster
}

struct RcGeom { int C, T, lgV, spc; size_t smem; };

bool rc_geometry(const ReconArgs& a, RcGeom& g) {
  static const int force = getenv("KMX_RECON_CLUSTER") ? atoi(getenv("KMX_RECON_CLUSTER")) : -1;
  if (force == 0 || a.carries || a.sequential || a.bias.enabled || a.dwords < 1 || a.dwords > 9) return false;
  const long long nstreams = (long long)a.batch * a.ns;
  int maxcount = a.s[0].count;
  if (a.ns > 1 && a.s[1].count > maxcount) maxcount = a.s[1].count;
  const int nsteps = maxcount - 1;
  if (nsteps < 64 || nstreams < 1) return false;
  // What one CTA per stream (k_recon_par) would have to stage: past its 216 KB the walks read
  // global memory step by step, and a cluster -- whose CTAs each stage a part -- wins at any
  // stream count (config 5, n = 8192, b = 128, ks2: 494 -> 146 us).  Streams that one CTA can
  // stage go to clusters only while there are too few of them to fill the chip (config 4).
  // (digits of at least 4 words: with narrower ones the unstaged walks keep up -- n = 8192, b = 32 / 64, ks2:
  // 52 / 86 us either way)
  const bool unstageable = a.dwords >= 4 &&
                           2 * ((size_t)(maxcount + 1) * a.dwords + (size_t)(maxcount + 1) / 8 + 1) * sizeof(u32) >
                               (size_t)216 * 1024;
  if (force < 0 && !unstageable && (nstreams * 2 > 148 || nsteps < 1024)) return false;
  int C = 2;
  if (force >= 2) {
    C = force > 8 ? 8 : force;
  } else {
    while (C < 8 && nstreams * (2 * C) <= 148 && nsteps / (2 * C) >= 512) C *= 2;
    if (unstageable && C < 4) C = 4;
  }
  static const int lgv0 = getenv("KMX_RECON_CL_LGV") ? atoi(getenv("KMX_RECON_CL_LGV")) : 3;
  for (; C <= 8; C *= 2) {
    for (int lgV = lgv0 < 1 ? 1 : lgv0; lgV <= 4; lgV++) {
      const int V = 1 << lgV;
      int T = ((nsteps + C - 1) / C + V - 1) / V;
      T = (T + 31) & ~31;
      if (T > RC_MAXT) continue;
      const int spc = T * V;
      const int nd = spc + 2;
      const size_t smem = 2 * ((size_t)nd * a.dwords + (nd >> lgV) + 1) * sizeof(u32);
      if (smem > 200 * 1024) continue;
      g.C = C; g.T = T; g.lgV = lgV; g.spc = spc; g.smem = smem;
      return true;
    }
    if (force >= 2) break;  // a forced cluster size is not widened
  }
  return false;
}

template <int NW>
cudaError_t rc_launch(const ReconArgs& a, const RcGeom& g, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_recon_cl<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((long long)a.batch * a.ns * g.C), 1, 1);
  cfg.blockDim = dim3((unsigned)g.T, 1, 1);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)g.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_recon_cl<NW>, a, g.lgV, g.spc);
}

}  // namespace

// A cluster per stream when the streams are few and long (or KMX_RECON_CLUSTER=C forces clusters
// of C; 0 disables); *used = false: not applicable, nothing launched.
cudaError_t launch_recon_cluster(const ReconArgs& a, cudaStream_t st, bool* used) {
  *used = false;
  RcGeom g;
  if (!rc_geometry(a, g)) return cudaSuccess;
  *used = true;
  switch (a.dwords) {
    case 1: return rc_launch<1>(a, g, st);
    case 2: return rc_launch<2>(a, g, st);
    case 3: return rc_launch<3>(a, g, st);
    case 4: return rc_launch<4>(a, g, st);
    case 5: return rc_launch<5>(a, g, st);
    case 6: return rc_launch<6>(a, g, st);
    case 7: return rc_launch<7>(a, g, st);
    case 8: return rc_launch<8>(a, g, st);
    default: return rc_launch<9>(a, g, st);
  }
}

}  // namespace kmx
