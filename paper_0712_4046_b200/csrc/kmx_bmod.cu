// kmx_bmod.cu -- bivariate R[x,y] -> R[x] reductions over R = Z/nZ
// (bipoly.py:177-278 with ring_zmod(n), :59-72), n word-sized.
//
// The same three phases as over Z (kmx_bivar.cu), in the ring's arithmetic:
//   k_bevalm     evaluation: y-chunks concatenated at a spacing, reversed
//                and/or with alternating signs, added mod n where they
//                overlap (_concat_chunks, bipoly.py:128-143)
//   univariate   the P products in (Z/nZ)[x] run through the integer KS
//                path itself (kmx_mod_mul: lift with b = bitlen(n-1), KS
//                product, K9 reduction) -- the multipoint substitution used
//                as the UniMul plug-in (bipoly.py:23)
//   k_brecoverm  half-sums with the ring's halving a * (n+1)/2 mod n (odd n
//                only, bipoly.py:64-66), the odd-part shift and the overlap
//                recovery (_overlap_recover :151-174, _split_chunks :146-148)
#include <cstring>
#include <mutex>

#include "../../include/kmx.h"
#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {
namespace {

struct ModN {
  u64 n;
  __device__ __forceinline__ u64 add(u64 a, u64 b) const {
    const u64 s = a + b;
    return (s < a || s >= n) ? s - n : s;
  }
  __device__ __forceinline__ u64 sub(u64 a, u64 b) const { return a >= b ? a - b : a + (n - b); }
  // a * (n+1)/2 mod n for odd n: a/2 if a is even, else (a+n)/2 (no overflow)
  __device__ __forceinline__ u64 halve(u64 a) const { return (a & 1) ? (a >> 1) + (n >> 1) + 1 : a >> 1; }
};

// evals: EF, EG [batch*P][Lu] u64 residues (product z = pair*P + point)
__global__ void __launch_bounds__(256) k_bevalm(BivarPlan p, ModN R, const u64* f, const u64* g, u64* ef,
                                                u64* eg, uint32_t* errx) {
  const int lx = p.lx, ly = p.ly, Lu = p.Lu, sp = p.spacing;
  const long long total = (long long)p.batch * p.P * 2 * Lu;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < total;
       id += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(id % Lu);
    long long r = id / Lu;
    const int side = (int)(r % 2);
    r /= 2;
    const int pt = (int)(r % p.P);
    const long long pair = r / p.P;
    int rev = 0, alt = 0;
    if (p.variant == 2) rev = pt == 1;
    else if (p.variant == 3) alt = pt == 1;
    else if (p.variant == 4) { alt = pt & 1; rev = (pt >> 1) & 1; }
    const u64* c = (side ? g : f) + pair * lx * ly;
    int qlo = t - lx + 1 <= 0 ? 0 : (t - lx + 1 + sp - 1) / sp;
    int qhi = t / sp;
    if (qhi > ly - 1) qhi = ly - 1;
    u64 acc = 0;
    for (int q = qlo; q <= qhi; q++) {
      const int k = rev ? (ly - 1 - q) : q;
      const u64 v = c[(long long)(t - q * sp) * ly + k];
      if (v >= R.n) raise_err(errx, ERR_INVAL);  // residues in [0, n)
      acc = (alt && (k & 1)) ? R.sub(acc, v) : R.add(acc, v);
    }
    (side ? eg : ef)[(pair * p.P + pt) * Lu + t] = acc;
  }
}

template <class FF, class RF>
__device__ void overlap_recover_m(const ModN& R, int count, int sp, int cl, int ybase, int ystep, int ly2, u64* H,
                                  FF fwd, RF rev) {
  const int low = min(sp, cl);
  const int ov = cl > sp ? cl - sp : 0;
  for (int t = threadIdx.x; t < low; t += blockDim.x) {
    u64 hi_prev = 0, lo_prev = 0;
    for (int k = 0; k < count; k++) {
      u64 lo = fwd((long long)k * sp + t);
      if (t < ov) lo = R.sub(lo, hi_prev);
      u64 hi = 0;
      if (t < ov) hi = R.sub(rev((long long)(count - 1 - k) * sp + sp + t), lo_prev);
      const int y = ybase + k * ystep;
      H[(long long)t * ly2 + y] = lo;
      if (t < ov) H[(long long)(sp + t) * ly2 + y] = hi;
      hi_prev = hi;
      lo_prev = lo;
    }
  }
}

// prods: [pair][P][2Lu-1] u64 residues; h: [pair][2lx-1][2ly-1]
__global__ void __launch_bounds__(128) k_brecoverm(BivarPlan p, ModN R, const u64* prods, u64* h,
                                                   const uint32_t* errx, uint32_t* err) {
  const int pair = blockIdx.x;
  if (pair == 0 && threadIdx.x == 0 && *errx) raise_err(err, *errx);  // the evaluation's input check
  const int lx = p.lx, ly = p.ly;
  const int lx2 = 2 * lx - 1, ly2 = 2 * ly - 1;
  const long long ps = 2LL * p.Lu - 1;
  const u64* pr = prods + (long long)pair * p.P * ps;
  u64* H = h + (long long)pair * lx2 * ly2;
  if (p.variant == 1) {  // bipoly.py:177-188
    const int sp = 2 * lx - 1;
    for (int id = threadIdx.x; id < lx2 * ly2; id += blockDim.x) {
      const int i = id / ly2, j = id - i * ly2;
      H[id] = pr[(long long)j * sp + i];
    }
  } else if (p.variant == 3) {  // bipoly.py:209-232
    const u64* pp = pr;
    const u64* pn = pr + ps;
    for (int id = threadIdx.x; id < lx2 * ly2; id += blockDim.x) {
      const int i = id / ly2, y = id - i * ly2;
      const int j = y >> 1;
      if ((y & 1) == 0) {
        const long long t = 2LL * lx * j + i;
        H[id] = R.halve(R.add(pp[t], pn[t]));
      } else {
        const long long t = 2LL * lx * j + i + lx;  // odd_vec = (...)[lx:]
        H[id] = R.halve(R.sub(pp[t], pn[t]));
      }
    }
  } else if (p.variant == 2) {  // bipoly.py:191-206
    const u64* pf = pr;
    const u64* pv = pr + ps;
    overlap_recover_m(R, 2 * ly - 1, lx, 2 * lx - 1, 0, 1, ly2, H, [&](long long x) { return pf[x]; },
                      [&](long long x) { return pv[x]; });
  } else {  // bipoly.py:235-278
    const int n = p.n4;
    const u64* pp = pr;
    const u64* pn = pr + ps;
    const u64* rp = pr + 2 * ps;
    const u64* rn = pr + 3 * ps;
    overlap_recover_m(R, ly, 2 * n, 2 * lx - 1, 0, 2, ly2, H,
                      [&](long long x) { return R.halve(R.add(pp[x], pn[x])); },
                      [&](long long x) { return R.halve(R.add(rp[x], rn[x])); });
    if (ly > 1)
      overlap_recover_m(R, ly - 1, 2 * n, 2 * lx - 1, 1, 2, ly2, H,
                        [&](long long x) { return R.halve(R.sub(pp[x + n], pn[x + n])); },
                        [&](long long x) { return R.halve(R.sub(rp[x + n], rn[x + n])); });
  }
}

int bmod_plan(BivarPlan& p, int variant, int batch, int lx, int ly, uint64_t n) {
  if (variant < 1 || variant > 4 || batch < 0 || lx < 1 || ly < 1 || n < 2) return KMX_EINVAL;
  if ((variant == 3 || variant == 4) && (n % 2) == 0) return KMX_EINVAL;  // MissingHalveError (bipoly.py:116-118)
  p.variant = variant; p.lx = lx; p.ly = ly; p.batch = batch;
  p.n4 = (lx + 1) / 2;
  switch (variant) {
    case 1: p.P = 1; p.spacing = 2 * lx - 1; p.Lu = (2 * lx - 1) * (ly - 1) + lx; break;
    case 2: p.P = 2; p.spacing = lx; p.Lu = lx * ly; break;
    case 3: p.P = 2; p.spacing = lx; p.Lu = lx * ly; break;
    default: p.P = 4; p.spacing = p.n4; p.Lu = p.n4 * (ly - 1) + lx; break;
  }
  return KMX_OK;
}

// KS variant for the univariate (Z/nZ)[x] products: the B200 AUTO bands
// (paper_0712_4046_b200.modpoly.GPU_THRESHOLDS, from the config-5 sweep)
int uni_variant(int Lu) { return Lu <= 64 ? 1 : (Lu <= 1024 ? 3 : 4); }

struct BmodLayout { size_t ws_mod, off_ef, off_eg, off_pr, total; };

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

BmodLayout bmod_layout(const BivarPlan& p, uint64_t n) {
  BmodLayout L;
  const long long nz = (long long)p.batch * p.P;
  // the KS workspace leads (its error word is the one kmx_ws_status reads)
  L.ws_mod = a256(kmx_mod_workspace_bytes(uni_variant(p.Lu), (int)nz, p.Lu, p.Lu, n));
  L.off_ef = L.ws_mod;
  L.off_eg = L.off_ef + a256((size_t)nz * p.Lu * 8);
  L.off_pr = L.off_eg + a256((size_t)nz * p.Lu * 8);
  L.total = L.off_pr + a256((size_t)nz * (2 * p.Lu - 1) * 8) + 256;  // + the evaluation's error word
  return L;
}

}  // namespace
}  // namespace kmx

using namespace kmx;

extern "C" {

size_t kmx_bks_mod_workspace_bytes(int variant, int batch, int lx, int ly, uint64_t modulus) {
  BivarPlan p;
  if (bmod_plan(p, variant, batch, lx, ly, modulus)) return 0;
  return bmod_layout(p, modulus).total;
}

int kmx_bks_mod_mul(int variant, int batch, int lx, int ly, uint64_t modulus, const uint64_t* f, const uint64_t* g,
                    uint64_t* h, void* workspace, size_t ws_bytes, void* stream) {
  BivarPlan p;
  int rc = bmod_plan(p, variant, batch, lx, ly, modulus);
  if (rc) return rc;
  const BmodLayout L = bmod_layout(p, modulus);
  if (ws_bytes < L.total || !workspace) return KMX_EINVAL;
  if (batch == 0) return KMX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  u64* ef = (u64*)(w + L.off_ef);
  u64* eg = (u64*)(w + L.off_eg);
  u64* pr = (u64*)(w + L.off_pr);
  ModN R{modulus};
  uint32_t* errx = (uint32_t*)(w + L.total - 256);
  if (cudaMemsetAsync(errx, 0, 4, st) != cudaSuccess) return KMX_ECUDA;
  const long long ne = (long long)batch * p.P * 2 * p.Lu;
  int grid = (int)((ne + 255) / 256 < 148LL * 32 ? (ne + 255) / 256 : 148LL * 32);
  if (grid < 1) grid = 1;
  k_bevalm<<<grid, 256, 0, st>>>(p, R, (const u64*)f, (const u64*)g, ef, eg, errx);
  if (cudaGetLastError() != cudaSuccess) return KMX_ECUDA;
  // univariate products in (Z/nZ)[x]: the KS path (pack -> multiply ->
  // finish [-> reconstruct] -> modular reduction); records its own kernels
  rc = kmx_mod_mul(uni_variant(p.Lu), batch * p.P, p.Lu, p.Lu, modulus, ef, eg, pr, w, L.ws_mod, stream);
  if (rc) return rc;
  const int nks = kmx_last_launch_count();
  k_brecoverm<<<batch, 128, 0, st>>>(p, R, pr, (u64*)h, errx, (uint32_t*)w);
  if (cudaGetLastError() != cudaSuccess) return KMX_ECUDA;
  g_launches = nks + 2;
  return KMX_OK;
}

int kmx_bks_mod_mul_host(int variant, int batch, int lx, int ly, uint64_t modulus, const uint64_t* f,
                         const uint64_t* g, uint64_t* h) {
  struct Ctx {
    std::mutex mu;
    cudaStream_t st = nullptr;
    void* buf[3] = {nullptr, nullptr, nullptr};
    size_t cap[3] = {0, 0, 0};
  };
  static Ctx ctx[16];
  BivarPlan p;
  int rc = bmod_plan(p, variant, batch, lx, ly, modulus);
  if (rc) return rc;
  if (batch == 0) return KMX_OK;
  const BmodLayout L = bmod_layout(p, modulus);
  const size_t fb = (size_t)batch * lx * ly * 8;
  const size_t hb = (size_t)batch * (2 * lx - 1) * (2 * ly - 1) * 8;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return KMX_ECUDA;
  Ctx& c = ctx[dev];
  std::lock_guard<std::mutex> lk(c.mu);
  if (!c.st && cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
  const size_t need[3] = {2 * a256(fb), hb, L.total};
  for (int i = 0; i < 3; i++) {
    if (c.cap[i] < need[i]) {
      if (c.buf[i]) cudaFree(c.buf[i]);
      c.buf[i] = nullptr;
      c.cap[i] = 0;
      const size_t want = need[i] > 4096 ? need[i] : 4096;
      if (cudaMalloc(&c.buf[i], want) != cudaSuccess) return KMX_ENOMEM;
      c.cap[i] = want;
    }
  }
  u64* dF = (u64*)c.buf[0];
  u64* dG = (u64*)((char*)c.buf[0] + a256(fb));
  if (cudaMemcpyAsync(dF, f, fb, cudaMemcpyHostToDevice, c.st) != cudaSuccess) return KMX_ECUDA;
  if (cudaMemcpyAsync(dG, g, fb, cudaMemcpyHostToDevice, c.st) != cudaSuccess) return KMX_ECUDA;
  rc = kmx_bks_mod_mul(variant, batch, lx, ly, modulus, dF, dG, (uint64_t*)c.buf[1], c.buf[2], c.cap[2], c.st);
  if (rc) return rc;
  if (cudaMemcpyAsync(h, c.buf[1], hb, cudaMemcpyDeviceToHost, c.st) != cudaSuccess) return KMX_ECUDA;
  return kmx_ws_status(c.buf[2], c.st);
}

}  // extern "C"
