// Bivariate R[x,y] -> R[x] reductions over R = Z (bipoly.py:177-278).
//
//   k_beval    evaluation: y-chunks concatenated at a spacing, optionally in
//              reversed chunk order and/or with alternating signs
//              (_concat_chunks, bipoly.py:128-143)
//   k_conv     batched univariate products in Z[x] (the UniMul plug-in,
//              bipoly.py:23, default uni_schoolbook oracle.py:58-69): int32 x
//              int32 -> int64 column sums, one IMAD.WIDE per product term
//   k_brecover half-sums, exact halving and the chunk overlap recovery
//              (_overlap_recover bipoly.py:151-174; _split_chunks :146-148)
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/kmx.h"
#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

// point descriptors: reverse / alternate flags per univariate product
struct BPoint { int reverse, alternate; };

__device__ __forceinline__ void point_flags(int variant, int pt, int& rev, int& alt) {
  rev = 0; alt = 0;
  if (variant == 2) rev = pt == 1;
  else if (variant == 3) alt = pt == 1;
  else if (variant == 4) { alt = pt & 1; rev = (pt >> 1) & 1; }
}

// evals: [2][batch * P][Lu] int32 (all f evaluations, then all g evaluations:
// each side is a contiguous [products][Lu] operand array for the KS path)
__global__ void __launch_bounds__(256) k_beval(BivarPlan p, const int32_t* f, const int32_t* g, int32_t* ev,
                                               uint32_t* err) {
  const int lx = p.lx, ly = p.ly, Lu = p.Lu, sp = p.spacing;
  const long long lim = 1LL << p.cbits;  // the declared bound the int64 budget was derived from
  bool bad = false;
  const long long total = (long long)p.batch * p.P * 2 * Lu;
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < total;
       id += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(id % Lu);
    long long r = id / Lu;
    const long long nprod = (long long)p.batch * p.P;
    const int side = (int)(r / nprod); r -= side * nprod;
    const int pt = (int)(r % p.P);
    const long long pair = r / p.P;
    int rev, alt;
    point_flags(p.variant, pt, rev, alt);
    const int32_t* c = (side ? g : f) + pair * lx * ly;
    // chunk positions q = (rev ? ly-1-k : k) with q*sp <= t < q*sp + lx
    int qlo = t - lx + 1 <= 0 ? 0 : (t - lx + 1 + sp - 1) / sp;
    int qhi = t / sp;
    if (qhi > ly - 1) qhi = ly - 1;
    long long acc = 0;
    for (int q = qlo; q <= qhi; q++) {
      const int k = rev ? (ly - 1 - q) : q;
      const int i = t - q * sp;
      const long long v = c[(long long)i * ly + k];
      bad |= v >= lim || v <= -lim;
      acc += (alt && (k & 1)) ? -v : v;
    }
    ev[id] = (int32_t)acc;
  }
  if (bad) raise_err(err, ERR_INVAL);
}

// Staged form (grids up to 48 KB): one CTA per (pair, side) loads the grid
// into shared memory with coalesced reads (the range check on the way) and
// evaluates every point from there -- the chunk walk reads the grid column-
// wise, which straight from global memory is one 4-byte access per line.
__global__ void __launch_bounds__(256) k_beval_s(BivarPlan p, const int32_t* f, const int32_t* g, int32_t* ev,
                                                 uint32_t* err) {
  extern __shared__ int32_t bs_grid[];
  const int lx = p.lx, ly = p.ly, Lu = p.Lu, sp = p.spacing;
  const long long pair = blockIdx.x >> 1;
  const int side = blockIdx.x & 1;
  const int32_t* c = (side ? g : f) + pair * lx * ly;
  const long long lim = 1LL << p.cbits;
  bool bad = false;
  for (int x = threadIdx.x; x < lx * ly; x += blockDim.x) {
    const int32_t v = __ldg(c + x);
    bad |= (long long)v >= lim || (long long)v <= -lim;
    bs_grid[x] = v;
  }
  if (bad) raise_err(err, ERR_INVAL);
  __syncthreads();
  const long long nprod = (long long)p.batch * p.P;
  for (int pt = 0; pt < p.P; pt++) {
    int rev, alt;
    point_flags(p.variant, pt, rev, alt);
    int32_t* out = ev + ((long long)side * nprod + pair * p.P + pt) * Lu;
    for (int t = threadIdx.x; t < Lu; t += blockDim.x) {
      const int qlo = t - lx + 1 <= 0 ? 0 : (t - lx + 1 + sp - 1) / sp;
      int qhi = t / sp;
      if (qhi > ly - 1) qhi = ly - 1;
      long long acc = 0;
      for (int q = qlo; q <= qhi; q++) {
        const int k = rev ? (ly - 1 - q) : q;
        const long long v = bs_grid[(t - q * sp) * ly + k];
        acc += (alt && (k & 1)) ? -v : v;
      }
      out[t] = (int32_t)acc;
    }
  }
}

// ------------------------------------------------------------ k_brecover
// One CTA per pair.  prods: [pair][P][p_stride] int64 (2Lu-1 valid).
// h: [pair][2lx-1][2ly-1] int64.
__device__ __forceinline__ long long halve(long long v, uint32_t* err) {
  if (v & 1) raise_err(err, ERR_INEXACT);  // bipoly.py:47-50
  return v >> 1;
}

// lanes t < min(sp, cl): sequential over chunks, chunk k -> output column
// y = ybase + k*ystep.  fwd(x) / rev(x) fetch the recovered-sum vectors.
// The per-row chains are independent: rows t are spread over the CTAs of
// the pair (blockIdx.y) and threads; each chain prefetches KB steps of its
// raw product words (loads only, no side effects, so they are all in flight
// together) before the dependent recurrence consumes them.
constexpr int BR_SPLIT = 4;  // CTAs per pair
template <bool HALVE, class FF, class RF>
__device__ void overlap_recover(int count, int sp, int cl, int ybase, int ystep, int ly2, int64_t* H, FF fwd,
                                RF rev, bool& odd, int t0, int tstride) {
  const int low = min(sp, cl);
  const int ov = cl > sp ? cl - sp : 0;
  constexpr int KB = 8;
  for (int t = t0; t < low; t += tstride) {
    long long hi_prev = 0, lo_prev = 0;  // high_{k-1}[t], low_{k-1}[t]
    const bool o = t < ov;
    for (int k0 = 0; k0 < count; k0 += KB) {
      long long f[KB], r[KB];
#pragma unroll
      for (int i = 0; i < KB; i++) {
        const int k = k0 + i;
        f[i] = k < count ? fwd((long long)k * sp + t) : 0;
        r[i] = (k < count && o) ? rev((long long)(count - 1 - k) * sp + sp + t) : 0;
      }
#pragma unroll
      for (int i = 0; i < KB; i++) {
        const int k = k0 + i;
        if (k >= count) break;
        long long fv = f[i], rv = r[i];
        if (HALVE) {  // the ring's halving (bipoly.py:47-50), exact over Z
          odd |= ((fv | rv) & 1) != 0;
          fv >>= 1;
          rv >>= 1;
        }
        long long lo = fv;
        long long hi = 0;
        if (o) {
          lo -= hi_prev;
          hi = rv - lo_prev;
        }
        const int y = ybase + k * ystep;
        H[(long long)t * ly2 + y] = lo;
        if (o) H[(long long)(sp + t) * ly2 + y] = hi;
        hi_prev = hi;
        lo_prev = lo;
      }
    }
  }
}

__global__ void __launch_bounds__(128) k_brecover(BivarPlan p, const int64_t* prods, long long p_stride,
                                                  int64_t* h, uint32_t* err, uint32_t* err0) {
  const int pair = blockIdx.x;
  // the KS products' error word leads the workspace (kmx_ws_status): fold the
  // evaluation's range check into it
  if (err0 && err0 != err && pair == 0 && blockIdx.y == 0 && threadIdx.x == 0 && *err) atomicOr(err0, *err);
  const int lx = p.lx, ly = p.ly;
  const int lx2 = 2 * lx - 1, ly2 = 2 * ly - 1;
  const int64_t* pr = prods + (long long)pair * p.P * p_stride;
  int64_t* H = h + (long long)pair * lx2 * ly2;
  bool odd = false;
  const int nthr = blockDim.x * gridDim.y;
  const int tid = blockIdx.y * blockDim.x + threadIdx.x;
  constexpr int U = 4;  // independent elements per thread in flight
  if (p.variant == 1 || p.variant == 3) {
    const int total = lx2 * ly2;
    const int64_t* pp = pr;
    const int64_t* pn = pr + p_stride;
    for (int base = tid; base < total; base += U * nthr) {
      long long a[U], c[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int id = base + u * nthr;
        a[u] = 0;
        c[u] = 0;
        if (id >= total) continue;
        const int i = id / ly2, y = id - i * ly2;
        if (p.variant == 1) {  // bipoly.py:177-188: split at spacing 2lx-1
          a[u] = __ldg(pr + (long long)y * (2 * lx - 1) + i);
        } else {  // bipoly.py:209-232: even y from the half-sum, odd y from the half-difference
          const int j = y >> 1;
          const long long t = 2LL * lx * j + i + ((y & 1) ? lx : 0);  // odd_vec = (...)[lx:]
          a[u] = __ldg(pp + t);
          c[u] = __ldg(pn + t);
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int id = base + u * nthr;
        if (id >= total) continue;
        long long v = a[u];
        if (p.variant == 3) {
          const int y = id % ly2;
          v = (y & 1) ? a[u] - c[u] : a[u] + c[u];
          odd |= (v & 1) != 0;
          v >>= 1;
        }
        H[id] = v;
      }
    }
  } else if (p.variant == 2) {  // bipoly.py:191-206
    const int64_t* pf = pr;
    const int64_t* pv = pr + p_stride;
    overlap_recover<false>(2 * ly - 1, lx, 2 * lx - 1, 0, 1, ly2, H,
                           [&](long long x) { return (long long)__ldg(pf + x); },
                           [&](long long x) { return (long long)__ldg(pv + x); }, odd, tid, nthr);
  } else {  // bipoly.py:235-278
    const int n = p.n4;
    const int64_t* pp = pr;
    const int64_t* pn = pr + p_stride;
    const int64_t* rp = pr + 2 * p_stride;
    const int64_t* rn = pr + 3 * p_stride;
    // the even and odd recoveries are independent: half the pair's CTAs each
    const int half = gridDim.y / 2 ? gridDim.y / 2 : 1;
    const int side = gridDim.y >= 2 ? (int)blockIdx.y / half : -1;  // -1: one CTA does both
    const int ht0 = (gridDim.y >= 2 ? (int)blockIdx.y % half : 0) * blockDim.x + threadIdx.x;
    const int hstride = half * blockDim.x;
    if (side != 1)
      overlap_recover<true>(ly, 2 * n, 2 * lx - 1, 0, 2, ly2, H,
                            [&](long long x) { return (long long)__ldg(pp + x) + __ldg(pn + x); },
                            [&](long long x) { return (long long)__ldg(rp + x) + __ldg(rn + x); }, odd, ht0,
                            hstride);
    if (ly > 1 && side != 0)
      overlap_recover<true>(ly - 1, 2 * n, 2 * lx - 1, 1, 2, ly2, H,
                            [&](long long x) { return (long long)__ldg(pp + x + n) - __ldg(pn + x + n); },
                            [&](long long x) { return (long long)__ldg(rp + x + n) - __ldg(rn + x + n); }, odd,
                            ht0, hstride);
  }
  if (odd) raise_err(err, ERR_INEXACT);  // inexact halving (bipoly.py:47-50)
}

static int getenv_b(const char* n, int d) {
  const char* v = getenv(n);
  return v && *v ? atoi(v) : d;
}

cudaError_t launch_bivar(const BivarPlan& p, const int32_t* f, const int32_t* g, int64_t* h, int32_t* evals,
                         int64_t* prods, uint32_t* err, cudaStream_t st, int* nlaunch, void* ks_ws,
                         size_t ks_ws_bytes, uint32_t* err0) {
  *nlaunch = 0;
  prof_reset();
  const long long nprod = (long long)p.batch * p.P;
  const long long ne = nprod * 2 * p.Lu;
  int grid = (int)std::min<long long>((ne + 255) / 256, 148LL * 32);
  if (grid < 1) grid = 1;
  prof_mark(0, true, st);
  const size_t gsm = (size_t)p.lx * p.ly * 4;
  if (gsm <= 48 * 1024 && getenv_b("KMX_BEVAL_STAGED", 1))
    k_beval_s<<<2 * p.batch, 256, gsm, st>>>(p, f, g, evals, err);
  else
    k_beval<<<grid, 256, 0, st>>>(p, f, g, evals, err);
  prof_mark(0, false, st);
  (*nlaunch)++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  long long ps;
  prof_mark(1, true, st);
  if (p.uni) {
    // univariate products on the integer KS path (Kronecker substitution of
    // the evaluations themselves): signed ebits-bit coefficients, int64
    // (two-word two's complement) product coefficients
    ps = 2LL * p.Lu - 1;
    const bool was = prof_suspend();
    const int rc = kmx_ks_mul(p.uni, (int)nprod, p.Lu, p.Lu, p.ebits, reinterpret_cast<const uint32_t*>(evals),
                              reinterpret_cast<const uint32_t*>(evals + nprod * p.Lu), 1,
                              reinterpret_cast<uint32_t*>(prods), 2, ks_ws, ks_ws_bytes, KMX_SIGNED, st);
    prof_resume(was);
    prof_keep(0);
    prof_keep(1);
    if (rc) return rc == KMX_ECUDA ? cudaErrorLaunchFailure : cudaErrorInvalidValue;
    *nlaunch += kmx_last_launch_count();
  } else {
    // univariate products (kmx_mul.cu)
    int split, cw, nbands, tr;
    mul_geometry(p.Lu, p.Lu, &split, &cw, &nbands, &tr);
    ps = (long long)nbands * cw;
    ConvArgs ca;
    ca.A = evals; ca.a_stride = p.Lu;
    ca.B = evals + nprod * p.Lu; ca.b_stride = p.Lu;
    ca.L = p.Lu;
    ca.P = prods; ca.p_stride = ps;
    ca.nprod = (int)nprod; ca.nbands = nbands; ca.G = split; ca.TI = tr;
    ca.counter = (int*)(err + 1);
    if ((e = launch_conv(ca, st)) != cudaSuccess) return e;
    (*nlaunch)++;
  }
  prof_mark(1, false, st);
  prof_mark(2, true, st);
  k_brecover<<<dim3(p.batch, BR_SPLIT), 128, 0, st>>>(p, prods, ps, h, err, err0);
  prof_mark(2, false, st);
  (*nlaunch)++;
  return cudaGetLastError();
}

}  // namespace kmx

// ------------------------------------------------------------------ C ABI
using namespace kmx;

namespace {
int env_int_b(const char* n, int d) {
  const char* v = getenv(n);
  return v && *v ? atoi(v) : d;
}

// Univariate product engine: the integer KS path when its product
// coefficients fit two words and the products are long enough for the tensor
// cores to pay, else k_conv.  Measured at c3 (256 pairs of 64x64 u16 grids,
// profiles/r02/bks_uni_c3.json): ks3 wins at Lu = 2080 and 4096 (1.57x /
// 2.4x over k_conv), ks4 at Lu = 8065 (2.9x).  KMX_BKS_UNI=0 forces k_conv,
// 1..4 a KS variant.
int bks_uni(const BivarPlan& p) {
  const int force = env_int_b("KMX_BKS_UNI", -1);
  if (force == 0) return 0;
  if (p.ebits > 32 || kmx_ks_out_words(p.Lu, p.Lu, p.ebits, KMX_SIGNED) != 2) return 0;
  if (force >= 1 && force <= 4) return force;
  if (p.Lu < env_int_b("KMX_BKS_KS_MIN", 512)) return 0;
  return p.Lu <= 4096 ? 3 : 4;
}

int bks_plan(BivarPlan& p, int variant, int batch, int lx, int ly, int coeff_bits) {
  if (variant < 1 || variant > 4 || batch < 0 || lx < 1 || ly < 1 || coeff_bits < 1 || coeff_bits > 30)
    return KMX_EINVAL;
  p.variant = variant; p.lx = lx; p.ly = ly; p.batch = batch;
  p.n4 = (lx + 1) / 2;
  p.cbits = coeff_bits;
  switch (variant) {
    case 1: p.P = 1; p.spacing = 2 * lx - 1; p.Lu = (2 * lx - 1) * (ly - 1) + lx; break;
    case 2: p.P = 2; p.spacing = lx; p.Lu = lx * ly; break;
    case 3: p.P = 2; p.spacing = lx; p.Lu = lx * ly; break;
    default: p.P = 4; p.spacing = p.n4; p.Lu = p.n4 * (ly - 1) + lx; break;
  }
  // |eval| < 2^(cb + [four-point overlap]); every univariate product
  // coefficient (and the half-sum numerators) must stay inside int64
  const int eb = coeff_bits + (variant == 4 ? 1 : 0);
  if (eb > 31) return KMX_EINVAL;
  double bound = (double)p.Lu * (double)(1ULL << eb) * (double)(1ULL << eb) * 2.0;
  if (bound >= 9.2e18) return KMX_EINVAL;
  p.ebits = eb + 1;  // two's-complement width of the evaluations
  p.uni = bks_uni(p);
  return KMX_OK;
}

size_t align256b(size_t x) { return (x + 255) & ~(size_t)255; }

struct BksLayout { size_t ks, err, ev, pr, total; };

// [KS workspace (its error word first: kmx_ws_status)] [error word + conv
// counter] [evaluations [2][B P][Lu]] [products]
BksLayout bks_layout(const BivarPlan& p) {
  BksLayout L;
  const long long nprod = (long long)p.batch * p.P;
  L.ks = p.uni ? align256b(kmx_ks_workspace_bytes(p.uni, (int)nprod, p.Lu, p.Lu, p.ebits, KMX_SIGNED)) : 0;
  size_t o = L.ks;
  L.err = o; o += 256;
  L.ev = o; o = align256b(o + (size_t)nprod * 2 * p.Lu * 4);
  long long ps;
  if (p.uni) {
    ps = 2LL * p.Lu - 1;
  } else {
    int split, cw, nbands, tr;
    mul_geometry(p.Lu, p.Lu, &split, &cw, &nbands, &tr);
    ps = (long long)nbands * cw;
  }
  L.pr = o; o = align256b(o + (size_t)nprod * ps * 8);
  L.total = o;
  return L;
}
}  // namespace

extern "C" {

size_t kmx_bks_workspace_bytes(int variant, int batch, int lx, int ly) {
  // the k_conv layout: valid for every coefficient bound
  BivarPlan p;
  if (bks_plan(p, variant, batch, lx, ly, 1)) return 0;
  p.uni = 0;
  return bks_layout(p).total;
}

int kmx_bks_uni_engine(int variant, int lx, int ly, int coeff_bits) {
  BivarPlan p;
  int rc = bks_plan(p, variant, 1, lx, ly, coeff_bits);
  return rc ? rc : p.uni;
}

size_t kmx_bks_workspace_bytes_cb(int variant, int batch, int lx, int ly, int coeff_bits) {
  BivarPlan p;
  if (bks_plan(p, variant, batch, lx, ly, coeff_bits)) return 0;
  return std::max(bks_layout(p).total, kmx_bks_workspace_bytes(variant, batch, lx, ly));
}

int kmx_bks_mul(int variant, int batch, int lx, int ly, int coeff_bits, const int32_t* f, const int32_t* g,
                int64_t* h, void* workspace, size_t ws_bytes, void* stream) {
  BivarPlan p;
  int rc = bks_plan(p, variant, batch, lx, ly, coeff_bits);
  if (rc) return rc;
  BksLayout L = bks_layout(p);
  if (ws_bytes < L.total && p.uni) {  // a workspace sized for k_conv only
    p.uni = 0;
    L = bks_layout(p);
  }
  if (ws_bytes < L.total) return KMX_EINVAL;
  if (batch == 0) return KMX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  uint32_t* err = (uint32_t*)(w + L.err);
  if (cudaMemsetAsync(err, 0, 8, st) != cudaSuccess) return KMX_ECUDA;  // error flag + work counter
  int nl = 0;
  cudaError_t e = launch_bivar(p, f, g, h, (int32_t*)(w + L.ev), (int64_t*)(w + L.pr), err, st, &nl,
                               p.uni ? w : nullptr, L.ks, (uint32_t*)w);
  g_launches = nl;
  if (e == cudaErrorInvalidValue) return KMX_EINVAL;
  return e == cudaSuccess ? KMX_OK : KMX_ECUDA;
}

int kmx_bks_mul_host(int variant, int batch, int lx, int ly, int coeff_bits, const int32_t* f, const int32_t* g,
                     int64_t* h) {
  // cached per-device buffers and stream (as kmx_ks_mul_host)
  struct Ctx {
    std::mutex mu;
    cudaStream_t st = nullptr;
    void* buf[3] = {nullptr, nullptr, nullptr};
    size_t cap[3] = {0, 0, 0};
  };
  static Ctx ctx[16];
  BivarPlan p;
  int rc = bks_plan(p, variant, batch, lx, ly, coeff_bits);
  if (rc) return rc;
  const size_t tot = kmx_bks_workspace_bytes_cb(variant, batch, lx, ly, coeff_bits);
  const size_t fb = (size_t)batch * lx * ly * 4;
  const size_t hb = (size_t)batch * (2 * lx - 1) * (2 * ly - 1) * 8;
  if (batch == 0) return KMX_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return KMX_ECUDA;
  Ctx& c = ctx[dev];
  std::lock_guard<std::mutex> lk(c.mu);
  if (!c.st && cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
  const size_t need[3] = {2 * align256b(fb), hb, tot};
  for (int i = 0; i < 3; i++) {
    if (c.cap[i] < need[i]) {
      if (c.buf[i]) cudaFree(c.buf[i]);
      c.buf[i] = nullptr;
      c.cap[i] = 0;
      if (cudaMalloc(&c.buf[i], need[i] > 4096 ? need[i] : 4096) != cudaSuccess) return KMX_ENOMEM;
      c.cap[i] = need[i] > 4096 ? need[i] : 4096;
    }
  }
  int32_t* dF = (int32_t*)c.buf[0];
  int32_t* dG = (int32_t*)((char*)c.buf[0] + align256b(fb));
  if (cudaMemcpyAsync(dF, f, fb, cudaMemcpyHostToDevice, c.st) != cudaSuccess) return KMX_ECUDA;
  if (cudaMemcpyAsync(dG, g, fb, cudaMemcpyHostToDevice, c.st) != cudaSuccess) return KMX_ECUDA;
  rc = kmx_bks_mul(variant, batch, lx, ly, coeff_bits, dF, dG, (int64_t*)c.buf[1], c.buf[2], c.cap[2], c.st);
  if (rc) return rc;
  if (cudaMemcpyAsync(h, c.buf[1], hb, cudaMemcpyDeviceToHost, c.st) != cudaSuccess) return KMX_ECUDA;
  return kmx_ws_status(c.buf[2], c.st);
}

}  // extern "C"
