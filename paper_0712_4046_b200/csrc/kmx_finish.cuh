// kmx_finish.cuh -- the warp-per-stream finish body (K3), shared by the
// standalone kernel k_finish_w (kmx_finish.cu: digits to the global digit
// buffer) and the fused finish + reconstruction kernel k_finrec (kmx_ks.cu:
// digits straight into the reconstruction's shared-memory stream copy).
// See kmx_finish.cu for the algorithm.
#pragma once

#include "kmx_common.cuh"
#include "kmx_internal.h"
#include "kmx_store.cuh"

namespace kmx {

constexpr int FW_WARPS = 4;
constexpr int FW_V = 8;
constexpr int FW_CH = 32 * FW_V;  // limbs per warp chunk

// Digit sinks for mode-1 (digit-buffer) streams: base() once per stream,
// then word w of digit idx goes to base[off(idx, w)].
struct GlobalDigitSink {  // the digit buffer in global memory (k_finish_w)
  const FinishArgs* a;
  __device__ __forceinline__ u32* base(const Stream& S, int pair) const {
    return a->dbuf + ((long long)pair * a->dslots_pair + S.dslot) * a->dslot_stride;
  }
  __device__ __forceinline__ long long off(long long idx, int w) const { return idx * a->dwords + w; }
};
struct SmemDigitSink {    // the reconstruction's padded shared-memory copy (k_finrec)
  u32* ptr;
  int dw, lgV;
  __device__ __forceinline__ u32* base(const Stream&, int) const { return ptr; }
  __device__ __forceinline__ long long off(long long idx, int w) const {
    return (long long)idx * dw + (idx >> lgV) + w;  // dpos(idx, dw, lgV) + w
  }
};

// Word w of the W-bit digit starting at bit lb >= 0 of a chunk buffer of
// FIN_HALO + FW_CH words (bits at or above W masked off).
__device__ __forceinline__ u32 dig_word(const u32* buf, int lb, int w, int W) {
  const int bit = lb + 32 * w, q = bit >> 5;
  const u32 lo = buf[q], hi = q + 1 < FIN_HALO + FW_CH ? buf[q + 1] : 0u;
  u32 x = __funnelshift_r(lo, hi, bit & 31);
  const int rem = W - 32 * w;
  if (rem < 32) x &= (1u << rem) - 1u;
  return x;
}

// One output stream (index si of pair `pair`) by one warp; buf: FIN_HALO +
// FW_CH words of this warp's shared memory (16-byte aligned).  Digit-buffer
// streams (mode 1) go to the sink.
// NC = false: the products were written by this kernel (the fused K2 + K3 of
// kmx_tcs.cu): plain loads instead of the read-only ld.global.nc path.
template <bool NC>
__device__ __forceinline__ uint4 fin_ld4(const uint4* p) {
  return NC ? __ldg(p) : *p;
}
template <class Sink, bool NC = true>
__device__ __forceinline__ void finish_warp_stream(const FinishArgs& a, int pair, int si, u32* buf, Sink sink) {
  const int lane = threadIdx.x & 31;
  const Stream S = si == 0 ? a.s[0] : (si == 1 ? a.s[1] : (si == 2 ? a.s[2] : a.s[3]));
  const long long zP = (long long)pair * a.nprod_pair + S.zP;
  const u32* Pp = a.P + zP * a.p_stride;
  const unsigned long long* spP = a.spill + zP * a.nbands * 2;
  const u32* Qp = nullptr;
  const unsigned long long* spQ = nullptr;
  int sg = 0;
  if (S.qsign) {
    const long long zQ = (long long)pair * a.nprod_pair + S.zQ;
    Qp = a.P + zQ * a.p_stride;
    spQ = a.spill + zQ * a.nbands * 2;
    const u32* mt = a.meta + (long long)pair * a.meta_per_pair;
    const u32 ngt = mt[2 * S.qmeta] ^ mt[2 * (S.qmeta + a.mf_slot_stride)];  // mul_signed: xor
    sg = ngt ? -S.qsign : S.qsign;
  }
  const long long off = S.off;
  const int W = S.W;
  const int Wd = (W + 31) >> 5;
  const long long E = off + (long long)S.cnt * W;
  const int lgC = 31 - __clz(a.band_cols);
  const int cmask = (1 << lgC) - 1;
  const int mp = a.mp;
  int Qd = mp + 1;
  const long long qe = (E + 31) / 32 + 1;
  if (qe > Qd) Qd = (int)qe;
  u32* hpair = a.h + (long long)pair * a.h_pair_stride;
  u32* dbase = S.mode == 1 ? sink.base(S, pair) : nullptr;
  buf[lane] = 0u;  // halo (FIN_HALO == 32)
  i64 cin_chunk = 0;  // carry + hi of the previous chunk's top limb
  bool bad = false;
  long long jl_next = 0;
  for (int q00 = 0; q00 < Qd; q00 += FW_CH) {
    const int q0 = q00 + lane * FW_V;
    u32 lo[FW_V];
    i64 hi[FW_V];
    {
      u32 pv[FW_V], qv[FW_V];
      i64 s0 = 0, s1 = 0;
      const bool full = q0 + FW_V <= mp;
      const bool bstart = q0 > 0 && q0 < mp && (q0 & cmask) == 0;
      const int bidx = (q0 >> lgC) - 1;
      if (full) {
        const uint4 x0 = fin_ld4<NC>(reinterpret_cast<const uint4*>(Pp + q0));
        const uint4 x1 = fin_ld4<NC>(reinterpret_cast<const uint4*>(Pp + q0) + 1);
        pv[0] = x0.x; pv[1] = x0.y; pv[2] = x0.z; pv[3] = x0.w; pv[4] = x1.x; pv[5] = x1.y; pv[6] = x1.z; pv[7] = x1.w;
      } else {
#pragma unroll
        for (int v = 0; v < FW_V; v++) pv[v] = q0 + v < mp ? Pp[q0 + v] : 0u;
      }
      if (bstart) { s0 = (i64)spP[bidx * 2]; s1 = (i64)spP[bidx * 2 + 1]; }
      if (sg) {
        if (full) {
          const uint4 x0 = fin_ld4<NC>(reinterpret_cast<const uint4*>(Qp + q0));
          const uint4 x1 = fin_ld4<NC>(reinterpret_cast<const uint4*>(Qp + q0) + 1);
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
    i64 hprev = __shfl_up_sync(0xffffffffu, hi[FW_V - 1], 1);
    if (lane == 0) hprev = cin_chunk;
    const i64 hlast = __shfl_sync(0xffffffffu, hi[FW_V - 1], 31);
    // local resolution with carry-in 0
    u32 d[FW_V];
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
    const int f1 = allF == 0xffffffffu ? 1 : 0, z1 = any == 0u ? 1 : 0;
    // carry map: cin -1 -> c - all0, 0 -> c, +1 -> c + allF, entry i = cout + 1 for cin = i - 1.
    // Held in two forms so that a composition is one PRMT: bytes (the table that is indexed)
    // and nibbles (the selector); x -> later(earlier(x)) = PRMT(later bytes, earlier nibbles).
    const u32 e0 = (u32)(c - z1 + 1), e1 = (u32)(c + 1), e2 = (u32)(c + f1 + 1);
    u32 incB = e0 | (e1 << 8) | (e2 << 16);
    u32 incN = e0 | (e1 << 4) | (e2 << 8);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 pmN = __shfl_up_sync(0xffffffffu, incN, o);
      const u32 nb = __byte_perm(incB, 0u, pmN);  // byte i = incB[pmN nibble i] (byte 3 unused)
      if (lane >= o) {
        incB = nb;
        incN = (nb & 0x3u) | ((nb >> 4) & 0x30u) | ((nb >> 8) & 0x300u);
      }
    }
    u32 excB = __shfl_up_sync(0xffffffffu, incB, 1);
    if (lane == 0) excB = 0x020100u;  // identity
    const u32 totB = __shfl_sync(0xffffffffu, incB, 31);
    int k = (int)((excB >> 8) & 0xffu) - 1;  // the preceding lanes' map at carry-in 0
    if (k) {  // ripple the carry-in through this lane's digits
#pragma unroll
      for (int v = 0; v < FW_V; v++) {
        const u32 old = d[v];
        d[v] = old + (u32)k;
        k = k > 0 ? (d[v] == 0u ? 1 : 0) : (k < 0 && old == 0u ? -1 : 0);
      }
    }
    cin_chunk = (i64)((int)((totB >> 8) & 0xffu) - 1) + hlast;
    // exactness checks (bits below off, bits at or above E), chunk-uniform branch
    if (32LL * q00 < off || 32LL * (q00 + FW_CH) > E) {
#pragma unroll
      for (int v = 0; v < FW_V; v++) {
        const long long bit0 = 32LL * (q0 + v);
        if (bit0 < off) {
          const long long nb = off - bit0;
          const u32 msk = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
          bad |= (d[v] & msk) != 0u;
        }
        if (bit0 + 32 > E && q0 + v < Qd) {
          const long long from = E - bit0;
          const u32 msk = from <= 0 ? 0xffffffffu : (0xffffffffu << from);
          bad |= (d[v] & msk) != 0u;
        }
      }
    }
    uint4* b4 = reinterpret_cast<uint4*>(buf + FIN_HALO + lane * FW_V);
    b4[0] = make_uint4(d[0], d[1], d[2], d[3]);
    b4[1] = make_uint4(d[4], d[5], d[6], d[7]);
    __syncwarp();
    // digits whose top bit falls inside this chunk
    const long long chi = 32LL * (q00 + FW_CH);
    // stream bit positions stay below 2^31 (products of < 2^26 limbs), so
    // 32-bit divisions
    // jl: first digit whose top bit lies at or above clo = the previous chunk's jh
    // (ceil((u + 1) / W) - 1 = floor(u / W) for u > 0), so one division per chunk
    const long long jl = jl_next;
    const int u = (int)(chi - off);
    long long jh = u <= 0 ? 0 : u / W;
    if (jh > S.cnt) jh = S.cnt;
    jl_next = jh;
    const long long base = off - 32LL * (q00 - FIN_HALO);
    if (W <= 32 * FIN_HALO) {
      // lean extraction: every digit handled here starts inside the halo or
      // the chunk (bit >= 0), so chunk-local 32-bit positions, one funnel
      // shift per word and no range tests
      const int ib = (int)(base + jl * W);
      const bool two = S.mode == 1 && a.dwords == 2 && Wd == 2;
      const u32 m1 = W >= 64 ? 0xffffffffu : ((1u << (W - 32)) - 1u);
      for (int jj = lane; jj < (int)(jh - jl); jj += 32) {
        const int j = (int)jl + jj;
        const int lb = ib + jj * W;
        if (S.mode == 0) {
          const long long kpos = S.pos0 + (long long)j * S.pstride;
          u32* dst = hpair + kpos * a.out_words;
          if (a.bias.enabled) {
            unsigned __int128 hp = 0;
            for (int w = 0; w < Wd && w < 4; w++) hp |= (unsigned __int128)dig_word(buf, lb, w, W) << (32 * w);
            store_coeff128(dst, a.out_words, hp, kpos, a.bias, pair);
          } else {
            for (int w = 0; w < a.out_words; w++) dst[w] = w < Wd ? dig_word(buf, lb, w, W) : 0u;
          }
        } else {
          const int idx = S.reversed ? (S.cnt - 1 - j) : j;
          u32* dp = dbase + sink.off(idx, 0);
          if (two) {  // 33..64-bit digits: three words, two funnel shifts
            const int q = lb >> 5, sb = lb & 31;
            const u32 w0 = buf[q], w1 = buf[q + 1], w2 = q + 2 < FIN_HALO + FW_CH ? buf[q + 2] : 0u;
            const u32 x0 = __funnelshift_r(w0, w1, sb), x1 = __funnelshift_r(w1, w2, sb) & m1;
            if ((reinterpret_cast<uintptr_t>(dp) & 7) == 0) {
              *reinterpret_cast<uint2*>(dp) = make_uint2(x0, x1);
            } else {
              dp[0] = x0;
              dp[1] = x1;
            }
          } else {
#pragma unroll 2
            for (int w = 0; w < a.dwords; w++) dp[w] = w < Wd ? dig_word(buf, lb, w, W) : 0u;
          }
        }
      }
    } else
    for (long long j = jl + lane; j < jh; j += 32) {
      const long long lb = base + j * W;
      if (S.mode == 0) {
        const long long kpos = S.pos0 + j * S.pstride;
        u32* dst = hpair + kpos * a.out_words;
        if (a.bias.enabled) {
          unsigned __int128 hp = 0;
          for (int w = 0; w < Wd && w < 4; w++) {
            u32 x = bits32(buf, FIN_HALO + FW_CH, lb + 32 * w);
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
            x = bits32(buf, FIN_HALO + FW_CH, lb + 32 * w);
            const int rem = W - 32 * w;
            if (rem < 32) x &= (1u << rem) - 1u;
          }
          dst[w] = x;
        }
      } else {
        const long long idx = S.reversed ? (S.cnt - 1 - j) : j;
        for (int w = 0; w < a.dwords; w++) {
          u32 x = 0u;
          if (w < Wd) {
            x = bits32(buf, FIN_HALO + FW_CH, lb + 32 * w);
            const int rem = W - 32 * w;
            if (rem < 32) x &= (1u << rem) - 1u;
          }
          dbase[sink.off(idx, w)] = x;
        }
      }
    }
    __syncwarp();
    buf[lane] = buf[FW_CH + lane];
    __syncwarp();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) raise_err(a.err, ERR_INEXACT);
  if (lane == 0 && cin_chunk != 0) raise_err(a.err, ERR_INEXACT);
}

}  // namespace kmx
