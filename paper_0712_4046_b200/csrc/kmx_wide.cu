// kmx_wide.cu -- the finish (K3) and reconstruction (K4) for digit widths
// past the fast kernels' register / halo budgets: W > 32 (FIN_HALO - 1) bits
// in the chunked finish, or reconstruction digits of more than 17 words.
// The reference takes any coefficient bound (pack.py:36-46, ksint.py:82-98),
// so these keep the drop-in's domain equal to it (b past ~490 bits).
//
//   numerator  the stream's P +- sgn(Q)|Q| (ksint.py:270-273, :320-335) as a
//              normalized limb array, by the linear-combination kernels of
//              kmx_kara.cu (device-side sign of Q from the pack metadata);
//   k_wdigits  bit-field gather of the W-bit digits at offset off (the exact
//              halving and >> N of halve_exact / shr_bits_exact, bignat.py:
//              265-269, 310-317, and _unpack_ints :431-450): one thread per
//              output word, plus a zero check of every bit below off and at
//              or above off + cnt W (ERR_INEXACT, as the reference raises);
//   k_wrecon   the overlap reconstruction (_reconstruct, ksint.py:137-179)
//              with multiword digits in global scratch, one thread per
//              stream: slow, exact, any width (ERR_RECON on inconsistency).
#include <cstring>

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

namespace {

// bits [bit, bit + 32) of a little-endian limb array of n limbs (zero past it)
__device__ __forceinline__ u32 bits32(const u32* T, long long n, long long bit) {
  const long long q = bit >> 5;
  const int r = (int)(bit & 31);
  const u32 lo = (q >= 0 && q < n) ? __ldg(T + q) : 0u;
  const u32 hi = (q + 1 >= 0 && q + 1 < n) ? __ldg(T + q + 1) : 0u;
  return r ? __funnelshift_r(lo, hi, r) : lo;
}

__global__ void __launch_bounds__(256) k_wdigits(WideDigitArgs a) {
  const Stream& S = a.s;
  const int Wd = (S.W + 31) / 32;
  const int ow = S.mode == 0 ? a.out_words : a.dwords;  // words written per digit
  const int nw = ow > Wd ? ow : Wd;                     // words visited (past ow: must be 0)
  const long long per_pair = (long long)S.cnt * nw;
  const long long total = per_pair * a.batch;
  bool bad = false;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < total;
       id += (long long)gridDim.x * blockDim.x) {
    const long long pair = id / per_pair;
    const long long r = id - pair * per_pair;
    const long long j = r / nw;
    const int w = (int)(r - j * nw);
    const u32* T = a.T + pair * a.t_stride;
    u32 v = 0u;
    if (w < Wd) {
      v = bits32(T, a.t_len, S.off + j * S.W + 32LL * w);
      const int rem = S.W - 32 * w;
      if (rem < 32) v &= (1u << rem) - 1u;
    }
    if (w >= ow) {
      bad |= v != 0u;
    } else if (S.mode == 0) {
      a.h[pair * a.h_pair_stride + (long long)(S.pos0 + j * S.pstride) * a.out_words + w] = v;
    } else {
      const long long idx = S.reversed ? S.cnt - 1 - j : j;
      a.dbuf[(pair * a.dslots_pair + S.dslot) * a.dslot_stride + idx * a.dwords + w] = v;
    }
  }
  // every bit of the numerator outside [off, off + cnt W) is zero
  const long long E = S.off + (long long)S.cnt * S.W;
  const long long tot2 = a.t_len * a.batch;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < tot2;
       id += (long long)gridDim.x * blockDim.x) {
    const long long pair = id / a.t_len, q = id - pair * a.t_len;
    const u32 x = __ldg(a.T + pair * a.t_stride + q);
    if (!x) continue;
    const long long b0 = 32 * q;
    u32 keep = 0xffffffffu;  // bits of limb q inside [off, E)
    if (b0 + 32 <= S.off || b0 >= E) keep = 0u;
    else {
      if (b0 < S.off) keep &= 0xffffffffu << (S.off - b0);
      if (b0 + 32 > E) keep &= 0xffffffffu >> (b0 + 32 - E);
    }
    bad |= (x & ~keep) != 0u;
  }
  if (bad) raise_err(a.err, ERR_INEXACT);
}

// ------------------------------------------------------------ multiword ops
// x - y - bin over n words, result into r (may alias x or y); borrow out
__device__ u32 w_sub(u32* r, const u32* x, const u32* y, u32 bin, int n) {
  u32 br = bin;
  for (int i = 0; i < n; i++) {
    const u64 t = (u64)x[i] - y[i] - br;
    r[i] = (u32)t;
    br = (u32)(t >> 63);
  }
  return br;
}
__device__ bool w_gt(const u32* x, const u32* y, int n) {
  for (int i = n - 1; i >= 0; i--)
    if (x[i] != y[i]) return x[i] > y[i];
  return false;
}
__device__ bool w_eq(const u32* x, const u32* y, int n) {
  for (int i = 0; i < n; i++)
    if (x[i] != y[i]) return false;
  return true;
}
__device__ bool w_is_mask(const u32* x, int n, u32 topmask) {  // x == 2^W - 1
  for (int i = 0; i < n - 1; i++)
    if (x[i] != 0xffffffffu) return false;
  return x[n - 1] == topmask;
}

// coefficient lo + 2^W hi into out_words words (bits past out_words must be 0)
__device__ bool w_store_coeff(u32* dst, int ow, const u32* lo, const u32* hi, int W, int n) {
  const int ws = W >> 5, bs = W & 31;
  bool ok = true;
  const int tot = 2 * n + 1;
  for (int w = 0; w < tot; w++) {
    u32 v = w < n ? lo[w] : 0u;
    // hi shifted left by W bits: word w gets hi bits from word (w - ws) and (w - ws - 1)
    const int k = w - ws;
    const u32 a0 = (k >= 0 && k < n) ? hi[k] : 0u;
    const u32 a1 = (k - 1 >= 0 && k - 1 < n) ? hi[k - 1] : 0u;
    v |= bs ? ((a0 << bs) | (a1 >> (32 - bs))) : a0;
    if (w < ow) dst[w] = v;
    else ok &= v == 0u;
  }
  for (int w = tot; w < ow; w++) dst[w] = 0u;
  return ok;
}

__global__ void __launch_bounds__(64) k_wrecon(ReconArgs a, u32* scratch) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)a.batch * a.ns) return;
  const long long pair = gid / a.ns;
  const int si = (int)(gid - pair * a.ns);
  const ReconStream R = si == 0 ? a.s[0] : a.s[1];
  const int n = a.dwords, W = a.W;
  const u32 topmask = (W & 31) ? ((1u << (W & 31)) - 1u) : 0xffffffffu;
  const int count = R.count;
  const u32* F = a.dbuf + (pair * a.dslots_pair + R.fslot) * a.dslot_stride;
  const u32* V = a.dbuf + (pair * a.dslots_pair + R.rslot) * a.dslot_stride;
  u32* lo_prev = scratch + gid * 4LL * n;  // lo[j-1]
  u32* lo_cur = lo_prev + n;               // lo[j]
  u32* hh = lo_cur + n;                    // hi[j]
  u32* zero = hh + n;
  for (int i = 0; i < n; i++) { lo_prev[i] = 0u; zero[i] = 0u; lo_cur[i] = F[i]; }
  u32* H = a.h + pair * a.h_pair_stride;
  uint8_t* car = a.carries ? a.carries + gid * (2LL * count + 1) : nullptr;
  u32 cf = 0u;
  if (car)
    for (int i = 0; i < 2 * count + 1; i++) car[i] = 0;
  bool bad = false, ok_out = true;
  for (int j = 0; j + 1 < count; j++) {
    const u32 cr = w_gt(lo_cur, V + (long long)(j + 1) * n, n) ? 1u : 0u;  // ksint.py:154
    if (car) car[count + 1 + j] = (uint8_t)cr;
    w_sub(hh, V + (long long)j * n, j ? lo_prev : zero, cr, n);
    hh[n - 1] &= topmask;
    bad |= w_is_mask(hh, n, topmask);
    // lo[j+1] = fwd[j+1] - h - cf (mod 2^W); the borrow is the next forward carry
    for (int i = 0; i < n; i++) lo_prev[i] = lo_cur[i];
    const u32 br = w_sub(lo_cur, F + (long long)(j + 1) * n, hh, cf, n);
    // borrow past 2^W: the word-level borrow, or the bits above W
    const u32 over = (topmask != 0xffffffffu) ? ((lo_cur[n - 1] & ~topmask) != 0u) : br;
    lo_cur[n - 1] &= topmask;
    cf = over ? 1u : 0u;
    if (car) car[j + 1] = (uint8_t)cf;
    ok_out &= w_store_coeff(H + (long long)(R.pos0 + (long long)j * R.pstride) * a.out_words, a.out_words, lo_prev,
                            hh, W, n);
  }
  // last coefficient and the consistency checks (ksint.py:165-177)
  w_sub(hh, V + (long long)(count - 1) * n, count >= 2 ? lo_prev : zero, 0u, n);
  hh[n - 1] &= topmask;
  bad |= w_is_mask(hh, n, topmask);
  bad |= !w_eq(lo_cur, V + (long long)count * n, n);
  {  // h + cf == fwd[count]
    u32 c = cf;
    const u32* top = F + (long long)count * n;
    for (int i = 0; i < n; i++) {
      const u64 t = (u64)hh[i] + c;
      bad |= (u32)t != top[i];
      c = (u32)(t >> 32);
    }
    bad |= c != 0u;
  }
  ok_out &= w_store_coeff(H + (long long)(R.pos0 + (long long)(count - 1) * R.pstride) * a.out_words, a.out_words,
                          lo_cur, hh, W, n);
  if (bad) raise_err(a.err, ERR_RECON);
  if (!ok_out) raise_err(a.err, ERR_INEXACT);
}

}  // namespace

cudaError_t launch_wide_digits(const WideDigitArgs& a, cudaStream_t st) {
  if (a.batch == 0) return cudaSuccess;
  const long long work = (long long)a.batch * (a.s.cnt * (long long)a.out_words + a.t_len);
  long long grid = (work + 255) / 256;
  if (grid > 148LL * 16) grid = 148LL * 16;
  if (grid < 1) grid = 1;
  k_wdigits<<<(unsigned)grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

size_t wide_recon_scratch_words(int batch, int ns, int dwords) { return (size_t)batch * ns * 4 * dwords; }

cudaError_t launch_wide_recon(const ReconArgs& a, u32* scratch, cudaStream_t st) {
  const long long n = (long long)a.batch * a.ns;
  if (n == 0) return cudaSuccess;
  k_wrecon<<<(unsigned)((n + 63) / 64), 64, 0, st>>>(a, scratch);
  return cudaGetLastError();
}

}  // namespace kmx
