// kmx_finish.cu -- K3 for short streams: one WARP per output digit stream
// (the same contract as k_finish in kmx_ks.cu: half-sum / half-difference
// P + s*Q with the band spills folded in, exact halving and shifts,
// W-bit digit extraction and the ERR_INEXACT checks; ksint.py:219-279,
// :305-345; bignat.py:265-274, :310-317, :431-450).
//
// Why a warp: at the BASELINE shapes a stream is a few hundred to a few
// thousand limbs (c2 ks4: 1218), so a 256-thread block with 2048-limb chunks
// idles most of its lanes and pays a block barrier per scan.  Here a warp
// walks its stream in 256-limb chunks (8 limbs per lane) with shuffles only,
// and the carry resolution is cheap:
//   * y_v = P_v + s Q_v (+ spill) is split y = lo + 2^32 hi and hi moved one
//     limb up (z_v = lo_v + hi_(v-1)), so every carry lies in {-1, 0, 1};
//   * each lane resolves its 8 limbs sequentially assuming carry-in 0, which
//     gives its carry-out c0 and digits D; a carry-in of +1 (-1) changes the
//     carry-out only if D is all ones (all zeros), so the lane's carry map is
//     (c0 - all0, c0, c0 + allF) -- three compares instead of a map per limb;
//   * one 5-step shuffle scan composes the lane maps; the lanes whose
//     carry-in is nonzero ripple it through their 8 digits.
// The normalized limbs go to a per-warp shared buffer (with a 32-word halo
// for digits straddling chunks) and the lanes extract digits from it.
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"
#include "kmx_finish.cuh"

namespace kmx {

namespace {

__global__ void __launch_bounds__(32 * FW_WARPS, 8) k_finish_w(FinishArgs a, long long nstreams) {
  __shared__ __align__(16) u32 sbuf[FW_WARPS][FIN_HALO + FW_CH];
  const int wid = threadIdx.x >> 5;
  const long long gs = (long long)blockIdx.x * FW_WARPS + wid;
  if (gs >= nstreams) return;  // warp-uniform
  const int pair = (int)(gs / a.ns);
  const int si = (int)(gs - (long long)pair * a.ns);
  finish_warp_stream(a, pair, si, sbuf[wid], GlobalDigitSink{&a});
}

// ------------------------------------------------------------------------
// Chunk-parallel finish: one warp per (stream, 256-limb chunk) instead of one
// warp walking a whole stream, for streams too long / too few to fill the chip
// (c2 ks1: 1024 streams of 4734 limbs).  Two kernels:
//   k_finmap   every chunk's carry map {-1,0,1} -> {-1,0,1} (the chunk's hi
//              carry-in is data-local: the hi word of limb q00-1's sum);
//   k_finchunk every chunk composes its predecessors' maps into its carry-in,
//              resolves its 256 limbs and the next 32 (the upper halo), and
//              extracts the digits that START inside it.
// ------------------------------------------------------------------------
struct FinCtx {
  Stream S;
  const u32* Pp;
  const u32* Qp;
  const unsigned long long* spP;
  const unsigned long long* spQ;
  int sg, W, Wd, lgC, cmask, mp, Qd;
  long long off, E;
  __device__ __forceinline__ void init(const FinishArgs& a, int pair, int si) {
    S = si == 0 ? a.s[0] : (si == 1 ? a.s[1] : (si == 2 ? a.s[2] : a.s[3]));
    const long long zP = (long long)pair * a.nprod_pair + S.zP;
    Pp = a.P + zP * a.p_stride;
    spP = a.spill + zP * a.nbands * 2;
    Qp = nullptr;
    spQ = nullptr;
    sg = 0;
    if (S.qsign) {
      const long long zQ = (long long)pair * a.nprod_pair + S.zQ;
      Qp = a.P + zQ * a.p_stride;
      spQ = a.spill + zQ * a.nbands * 2;
      const u32* mt = a.meta + (long long)pair * a.meta_per_pair;
      const u32 ngt = mt[2 * S.qmeta] ^ mt[2 * (S.qmeta + a.mf_slot_stride)];  // mul_signed: xor
      sg = ngt ? -S.qsign : S.qsign;
    }
    off = S.off;
    W = S.W;
    Wd = (W + 31) >> 5;
    E = off + (long long)S.cnt * W;
    lgC = 31 - __clz(a.band_cols);
    cmask = (1 << lgC) - 1;
    mp = a.mp;
    Qd = mp + 1;
    const long long qe = (E + 31) / 32 + 1;
    if (qe > Qd) Qd = (int)qe;
  }
  // hi word of limb q's sum (0 outside [0, mp)); limb q is never a band start here
  __device__ __forceinline__ i64 hi1(int q) const {
    if (q < 0 || q >= mp) return 0;
    i64 y = (i64)Pp[q];
    if (sg > 0) y += (i64)Qp[q];
    else if (sg < 0) y -= (i64)Qp[q];
    const int r = q & cmask, bnd = q >> lgC;
    if (bnd > 0 && r < 2) {
      y += (i64)spP[(bnd - 1) * 2 + r];
      if (sg) y += sg * (i64)spQ[(bnd - 1) * 2 + r];
    }
    return y >> 32;
  }
  // limbs q0 .. q0+7 of P + s Q with the band spills, split into lo / hi
  __device__ __forceinline__ void load8(int q0, u32 lo[FW_V], i64 hi[FW_V]) const {
    u32 pv[FW_V], qv[FW_V];
    i64 s0 = 0, s1 = 0;
    const bool full = q0 + FW_V <= mp;
    const bool bstart = q0 > 0 && q0 < mp && (q0 & cmask) == 0;
    const int bidx = (q0 >> lgC) - 1;
    if (full) {
      const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(Pp + q0));
      const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(Pp + q0) + 1);
      pv[0] = x0.x; pv[1] = x0.y; pv[2] = x0.z; pv[3] = x0.w; pv[4] = x1.x; pv[5] = x1.y; pv[6] = x1.z; pv[7] = x1.w;
    } else {
#pragma unroll
      for (int v = 0; v < FW_V; v++) pv[v] = q0 + v < mp ? Pp[q0 + v] : 0u;
    }
    if (bstart) { s0 = (i64)spP[bidx * 2]; s1 = (i64)spP[bidx * 2 + 1]; }
    if (sg) {
      if (full) {
        const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(Qp + q0));
        const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(Qp + q0) + 1);
        qv[0] = x0.x; qv[1] = x0.y; qv[2] = x0.z; qv[3] = x0.w; qv[4] = x1.x; qv[5] = x1.y; qv[6] = x1.z; qv[7] = x1.w;
      } else {
#pragma unroll
        for (int v = 0; v < FW_V; v++) qv[v] = q0 + v < mp ? Qp[q0 + v] : 0u;
      }
      if (bstart) { s0 += sg * (i64)spQ[bidx * 2]; s1 += sg * (i64)spQ[bidx * 2 + 1]; }
    }
#pragma unroll
    for (int v = 0; v < FW_V; v++) {
      i64 y = (i64)pv[v];
      if (sg > 0) y += (i64)qv[v];
      else if (sg < 0) y -= (i64)qv[v];
      if (v == 0) y += s0;
      if (v == 1) y += s1;
      lo[v] = (u32)y;
      hi[v] = y >> 32;
    }
  }
};

// Thread-level resolution of 8 limbs with carry-in 0 (z_v = lo_v + hi_(v-1),
// hprev for v = 0): digits d and the 6-bit map (c0 - all0, c0, c0 + allF).
__device__ __forceinline__ u32 fin_local(const u32 lo[FW_V], const i64 hi[FW_V], i64 hprev, u32 d[FW_V]) {
  int c = 0;
  u32 allF = 0xffffffffu, any = 0u;
#pragma unroll
  for (int v = 0; v < FW_V; v++) {
    const i64 t = (i64)lo[v] + (v ? hi[v - 1] : hprev) + c;
    d[v] = (u32)t;
    c = (int)(t >> 32);
    allF &= d[v];
    any |= d[v];
  }
  return (u32)(c - (any == 0u ? 1 : 0) + 1) | ((u32)(c + 1) << 2) | ((u32)(c + (allF == 0xffffffffu ? 1 : 0) + 1) << 4);
}

__device__ __forceinline__ void fin_ripple(u32 d[FW_V], int k) {
  if (!k) return;
#pragma unroll
  for (int v = 0; v < FW_V; v++) {
    const u32 old = d[v];
    d[v] = old + (u32)k;
    k = k > 0 ? (d[v] == 0u ? 1 : 0) : (k < 0 && old == 0u ? -1 : 0);
  }
}

__device__ __forceinline__ long long fin_nstreams(const FinishArgs& a, int batch) { return (long long)batch * a.ns; }

__global__ void __launch_bounds__(32 * FW_WARPS) k_finmap(FinishArgs a, long long nunits) {
  const int lane = threadIdx.x & 31;
  const long long u = (long long)blockIdx.x * FW_WARPS + (threadIdx.x >> 5);
  if (u >= nunits) return;
  const long long gs = u / a.nchunks;
  const int c = (int)(u - gs * a.nchunks);
  const int pair = (int)(gs / a.ns), si = (int)(gs - (long long)pair * a.ns);
  FinCtx F;
  F.init(a, pair, si);
  const int q00 = c * FW_CH;
  if (q00 >= F.Qd) return;
  u32 lo[FW_V], d[FW_V];
  i64 hi[FW_V];
  F.load8(q00 + lane * FW_V, lo, hi);
  i64 hprev = __shfl_up_sync(0xffffffffu, hi[FW_V - 1], 1);
  if (lane == 0) hprev = F.hi1(q00 - 1);
  u32 inc = fin_local(lo, hi, hprev, d);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 pm = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = cm_compose(pm, inc);
  }
  if (lane == 31) a.cmaps[u] = (uint8_t)inc;
}

__global__ void __launch_bounds__(32 * FW_WARPS) k_finchunk(FinishArgs a, long long nunits) {
  const GlobalDigitSink sink{&a};  // built on the device: it points at this kernel's parameter
  __shared__ __align__(16) u32 sbuf[FW_WARPS][FW_CH + FIN_HALO];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long u = (long long)blockIdx.x * FW_WARPS + wid;
  if (u >= nunits) return;
  u32* buf = sbuf[wid];
  const long long gs = u / a.nchunks;
  const int c = (int)(u - gs * a.nchunks);
  const int pair = (int)(gs / a.ns), si = (int)(gs - (long long)pair * a.ns);
  FinCtx F;
  F.init(a, pair, si);
  const int q00 = c * FW_CH;
  if (q00 >= F.Qd) return;
  // carry into this chunk: the predecessors' maps composed, applied to 0
  int cin = 0;
  if (c > 0) {
    const uint8_t* mp_ = a.cmaps + gs * a.nchunks;
    const int per = (c + 31) >> 5;
    const int j0 = lane * per, j1 = min(c, j0 + per);
    u32 m = CM_IDENT;
    for (int j = j0; j < j1; j++) m = cm_compose(m, (u32)mp_[j]);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 pm = __shfl_up_sync(0xffffffffu, m, o);
      if (lane >= o) m = cm_compose(pm, m);
    }
    cin = cm_apply(__shfl_sync(0xffffffffu, m, 31), 0);
  }
  // this chunk: 256 limbs
  u32 lo[FW_V], d[FW_V];
  i64 hi[FW_V];
  F.load8(q00 + lane * FW_V, lo, hi);
  i64 hprev = __shfl_up_sync(0xffffffffu, hi[FW_V - 1], 1);
  if (lane == 0) hprev = F.hi1(q00 - 1);
  const i64 hlast = __shfl_sync(0xffffffffu, hi[FW_V - 1], 31);
  u32 inc = fin_local(lo, hi, hprev, d);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 pm = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = cm_compose(pm, inc);
  }
  u32 exc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) exc = CM_IDENT;
  const int cout = cm_apply(__shfl_sync(0xffffffffu, inc, 31), cin);
  fin_ripple(d, cm_apply(exc, cin));
  bool bad = false;
  if (32LL * q00 < F.off || 32LL * (q00 + FW_CH) > F.E) {
    const int q0 = q00 + lane * FW_V;
#pragma unroll
    for (int v = 0; v < FW_V; v++) {
      const long long bit0 = 32LL * (q0 + v);
      if (bit0 < F.off) {
        const long long nb = F.off - bit0;
        const u32 msk = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
        bad |= (d[v] & msk) != 0u;
      }
      if (bit0 + 32 > F.E && q0 + v < F.Qd) {
        const long long from = F.E - bit0;
        const u32 msk = from <= 0 ? 0xffffffffu : (0xffffffffu << from);
        bad |= (d[v] & msk) != 0u;
      }
    }
  }
  uint4* b4 = reinterpret_cast<uint4*>(buf + lane * FW_V);
  b4[0] = make_uint4(d[0], d[1], d[2], d[3]);
  b4[1] = make_uint4(d[4], d[5], d[6], d[7]);
  // upper halo: the next 32 limbs (lanes 0..3), carry-in = this chunk's carry-out
  if (lane < 4) {
    u32 hl[FW_V], hd[FW_V];
    i64 hh[FW_V];
    F.load8(q00 + FW_CH + lane * FW_V, hl, hh);
    i64 hp = __shfl_up_sync(0xfu, hh[FW_V - 1], 1, 4);
    if (lane == 0) hp = hlast;
    u32 hm = fin_local(hl, hh, hp, hd);
    for (int o = 1; o < 4; o <<= 1) {
      const u32 pm = __shfl_up_sync(0xfu, hm, o, 4);
      if (lane >= o) hm = cm_compose(pm, hm);
    }
    u32 he = __shfl_up_sync(0xfu, hm, 1, 4);
    if (lane == 0) he = CM_IDENT;
    fin_ripple(hd, cm_apply(he, cout));
    uint4* h4 = reinterpret_cast<uint4*>(buf + FW_CH + lane * FW_V);
    h4[0] = make_uint4(hd[0], hd[1], hd[2], hd[3]);
    h4[1] = make_uint4(hd[4], hd[5], hd[6], hd[7]);
  }
  __syncwarp();
  // the value carried past the stream must vanish (last chunk)
  if (q00 + FW_CH >= F.Qd && lane == 0 && (i64)cout + hlast != 0) bad = true;
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_err(a.err, ERR_INEXACT);
  // digits starting in [32 q00, 32 (q00 + 256))
  const long long clo = 32LL * q00 - F.off, chi = 32LL * (q00 + FW_CH) - F.off;
  long long jl = clo <= 0 ? 0 : (clo + F.W - 1) / F.W;
  long long jh = chi <= 0 ? 0 : (chi + F.W - 1) / F.W;
  if (jh > F.S.cnt) jh = F.S.cnt;
  const long long base = F.off - 32LL * q00;
  u32* hpair = a.h + (long long)pair * a.h_pair_stride;
  u32* dbase = F.S.mode == 1 ? sink.base(F.S, pair) : nullptr;
  const int W = F.W, Wd = F.Wd;
  if (W <= 32 * FIN_HALO) {
    // lean extraction (as finish_warp_stream): chunk-local 32-bit positions,
    // one funnel shift per word; digits start inside the chunk and end in
    // the upper halo at the latest
    const int ib = (int)(base + jl * W);
    for (int jj = lane; jj < (int)(jh - jl); jj += 32) {
      const int j = (int)jl + jj;
      const int lb = ib + jj * W;
      if (F.S.mode == 0) {
        const long long kpos = F.S.pos0 + (long long)j * F.S.pstride;
        u32* dst = hpair + kpos * a.out_words;
        if (a.bias.enabled) {
          unsigned __int128 hp = 0;
          for (int w = 0; w < Wd && w < 4; w++) hp |= (unsigned __int128)dig_word(buf, lb, w, W) << (32 * w);
          store_coeff128(dst, a.out_words, hp, kpos, a.bias, pair);
        } else {
          for (int w = 0; w < a.out_words; w++) dst[w] = w < Wd ? dig_word(buf, lb, w, W) : 0u;
        }
      } else {
        const int idx = F.S.reversed ? (F.S.cnt - 1 - j) : j;
        u32* dp = dbase + sink.off(idx, 0);
        for (int w = 0; w < a.dwords; w++) dp[w] = w < Wd ? dig_word(buf, lb, w, W) : 0u;
      }
    }
    return;
  }
  for (long long j = jl + lane; j < jh; j += 32) {
    const long long lb = base + j * W;
    if (F.S.mode == 0) {
      const long long kpos = F.S.pos0 + j * F.S.pstride;
      u32* dst = hpair + kpos * a.out_words;
      if (a.bias.enabled) {
        unsigned __int128 hp = 0;
        for (int w = 0; w < Wd && w < 4; w++) {
          u32 x = bits32(buf, FW_CH + FIN_HALO, lb + 32 * w);
          const int rem = W - 32 * w;
          if (rem < 32) x &= (1u << rem) - 1u;
          hp |= (unsigned __int128)x << (32 * w);
        }
        store_coeff128(dst, a.out_words, hp, kpos, a.bias, pair);
        continue;
      }
      for (int w = 0; w < a.out_words; w++) {
        u32 x = 0u;
        if (w < Wd) {
          x = bits32(buf, FW_CH + FIN_HALO, lb + 32 * w);
          const int rem = W - 32 * w;
          if (rem < 32) x &= (1u << rem) - 1u;
        }
        dst[w] = x;
      }
    } else {
      const long long idx = F.S.reversed ? (F.S.cnt - 1 - j) : j;
      for (int w = 0; w < a.dwords; w++) {
        u32 x = 0u;
        if (w < Wd) {
          x = bits32(buf, FW_CH + FIN_HALO, lb + 32 * w);
          const int rem = W - 32 * w;
          if (rem < 32) x &= (1u << rem) - 1u;
        }
        dbase[sink.off(idx, w)] = x;
      }
    }
  }
}

}  // namespace

// Chunk-parallel finish (k_finmap + k_finchunk) when the warp-per-stream
// kernel would leave the chip short of warps relative to the chunk count;
// KMX_FINISH_CHUNKS=0/1 forces.
bool finish_use_chunks(const FinishArgs& a, int batch) {
  static const int force = getenv("KMX_FINISH_CHUNKS") ? atoi(getenv("KMX_FINISH_CHUNKS")) : -1;
  if (!a.cmaps || a.nchunks < 1) return false;
  if (force >= 0) return force != 0;
  // it does ~2x the carry work of the warp-per-stream kernel, so it pays only
  // for few, long streams (c4: 32-128 streams of 67-134 chunks, ks1 finish
  // 131 -> 33 us); at c1/c2 (>= 64 streams of <= 19 chunks) it is 10-50% slower
  const long long streams = (long long)batch * a.ns;
  return a.nchunks >= 16 && streams < 512;
}

// Warp-per-stream finish when streams are short (few chunks each) or there
// are enough of them to fill the chip with warps; KMX_FINISH_WARP=0/1 forces.
// The chunk-parallel variant rides on the same switch.
bool finish_use_warp(const FinishArgs& a, int batch) {
  static const int force = getenv("KMX_FINISH_WARP") ? atoi(getenv("KMX_FINISH_WARP")) : -1;
  if (force >= 0) return force != 0;
  if (finish_use_chunks(a, batch)) return true;
  const long long streams = (long long)batch * a.ns;
  return a.mp <= 1024 || (a.mp <= 8192 && streams >= 148LL * 8);
}

cudaError_t launch_finish_w(const FinishArgs& a, int batch, cudaStream_t st) {
  const long long ns = (long long)batch * a.ns;
  if (finish_use_chunks(a, batch)) {
    const long long nu = ns * a.nchunks;
    const long long blocks = (nu + FW_WARPS - 1) / FW_WARPS;
    k_finmap<<<(unsigned)blocks, 32 * FW_WARPS, 0, st>>>(a, nu);
    k_finchunk<<<(unsigned)blocks, 32 * FW_WARPS, 0, st>>>(a, nu);
    return cudaGetLastError();
  }
  const long long blocks = (ns + FW_WARPS - 1) / FW_WARPS;
  k_finish_w<<<(unsigned)blocks, 32 * FW_WARPS, 0, st>>>(a, ns);
  return cudaGetLastError();
}

}  // namespace kmx
