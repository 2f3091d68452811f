// kmx_bwide.cu -- the bivariate reductions over R = Z for coefficients of any
// width (bipoly.py:177-278 with ring_z(), :53-56: the reference takes any
// integer), beyond the int32-input / int64-accumulation kernels of
// kmx_bivar.cu.
//
// The reduction runs, unchanged, over R = Z/p for k word-sized primes p_i
// (each one kmx_bks_mod_mul: the same evaluation, the univariate products on
// the integer KS path, the half-sums with the ring's halving and the overlap
// recovery, bipoly.py:59-72), and the coefficients over Z are recovered by
// CRT: prod p_i > 2 max|h| with |h| < lx ly 2^(2 coeff_bits).  Halving mod an
// odd p agrees with exact halving over Z because the Z values being halved
// are even (the reductions' own invariant).
//
//   k_wres    signed multiword inputs -> residues mod every p_i, with the
//             |c| < 2^coeff_bits range check (ERR_INVAL);
//   k_garner  per output coefficient: mixed-radix digits of its residues
//             (Garner), the value as a multiword integer, the symmetric
//             representative in (-P/2, P/2], two's complement out.
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/kmx.h"
#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {
namespace {

constexpr int BW_KMAX = 16;             // primes (bound bits up to 16 * 61)
constexpr int BW_PW = 2 * BW_KMAX + 2;  // u32 words of the CRT modulus

struct CrtParams {
  u64 p[BW_KMAX];
  u64 inv[BW_KMAX][BW_KMAX];  // inv[j][i] = p_j^-1 mod p_i (j < i)
  u32 P[BW_PW];               // prod p_i
  int k, pw;
};

__host__ __device__ inline u64 mulmod(u64 a, u64 b, u64 m) { return (u64)((unsigned __int128)a * b % m); }

u64 powmod_h(u64 a, u64 e, u64 m) {
  u64 r = 1 % m;
  a %= m;
  while (e) {
    if (e & 1) r = mulmod(r, a, m);
    a = mulmod(a, a, m);
    e >>= 1;
  }
  return r;
}
bool is_prime_u64(u64 n) {  // deterministic Miller-Rabin for 64-bit n
  if (n < 2) return false;
  for (u64 q : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull})
    if (n % q == 0) return n == q;
  u64 d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; s++; }
  for (u64 a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    u64 x = powmod_h(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; r++) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}

// the BW_KMAX largest primes below 2^62
const std::vector<u64>& primes() {
  static std::vector<u64> v;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (v.empty())
    for (u64 n = (1ull << 62) - 1; (int)v.size() < BW_KMAX; n -= 2)
      if (is_prime_u64(n)) v.push_back(n);
  return v;
}

int bound_bits(int lx, int ly, int cb) {  // |h| < lx ly 2^(2 cb)
  int lg = 0;
  while ((1ll << lg) < (long long)lx * ly) lg++;
  return 2 * cb + lg;
}
int nprimes(int lx, int ly, int cb) { return (bound_bits(lx, ly, cb) + 2 + 60) / 61; }  // p_i > 2^61

bool crt_params(int k, CrtParams& c) {
  if (k < 1 || k > BW_KMAX) return false;
  memset(&c, 0, sizeof c);
  const std::vector<u64>& ps = primes();
  c.k = k;
  for (int i = 0; i < k; i++) c.p[i] = ps[i];
  for (int i = 0; i < k; i++)
    for (int j = 0; j < i; j++) c.inv[j][i] = powmod_h(c.p[j] % c.p[i], c.p[i] - 2, c.p[i]);
  // P = prod p_i in u32 words
  c.P[0] = 1;
  int n = 1;
  for (int i = 0; i < k; i++) {
    unsigned __int128 carry = 0;
    for (int w = 0; w < n; w++) {
      const unsigned __int128 t = (unsigned __int128)c.P[w] * c.p[i] + carry;
      c.P[w] = (u32)t;
      carry = t >> 32;
    }
    while (carry) { c.P[n++] = (u32)carry; carry >>= 32; }
  }
  c.pw = n;
  return true;
}

__global__ void __launch_bounds__(256) k_wres(CrtParams c, const u32* x, long long count, int iw, int cb, u64* res,
                                              long long res_stride, u32* err) {
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < count;
       id += (long long)gridDim.x * blockDim.x) {
    const u32* v = x + id * iw;
    const bool neg = (v[iw - 1] >> 31) != 0;
    // |c| word by word (two's complement negation on the fly) and the range check
    bool bad = false;
    u32 cy = 1;
    // magnitude words low to high, then Horner from the top word per prime
    u32 mag[64];
    for (int w = 0; w < iw && w < 64; w++) {
      u32 m = v[w];
      if (neg) {
        const u64 t = (u64)(~m) + cy;
        m = (u32)t;
        cy = (u32)(t >> 32);
      }
      mag[w] = m;
      const int lo = 32 * w;
      if (lo + 32 > cb) {  // bits at or above cb must be zero
        const u32 keep = cb > lo ? ((cb - lo >= 32) ? 0xffffffffu : ((1u << (cb - lo)) - 1u)) : 0u;
        bad |= (m & ~keep) != 0u;
      }
    }
    for (int i = 0; i < c.k; i++) {
      const u64 p = c.p[i];
      u64 acc = 0;
      for (int w = iw - 1; w >= 0; w--) acc = (u64)((((unsigned __int128)acc << 32) + mag[w]) % p);
      if (neg && acc) acc = p - acc;
      res[i * res_stride + id] = acc;
    }
    if (bad) raise_err(err, ERR_INVAL);
  }
}

__global__ void __launch_bounds__(128) k_garner(CrtParams c, const u64* res, long long res_stride, long long count,
                                                u32* h, int ow) {
  for (long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x; id < count;
       id += (long long)gridDim.x * blockDim.x) {
    u64 a[BW_KMAX];
    for (int i = 0; i < c.k; i++) {
      const u64 p = c.p[i];
      u64 t = res[i * res_stride + id] % p;
      for (int j = 0; j < i; j++) {
        const u64 aj = a[j] % p;
        t = t >= aj ? t - aj : t + p - aj;
        t = mulmod(t, c.inv[j][i], p);
      }
      a[i] = t;
    }
    // x = a_0 + p_0 (a_1 + p_1 (a_2 + ...)), Horner from the top
    u32 x[BW_PW];
    for (int w = 0; w < BW_PW; w++) x[w] = 0u;
    int n = 0;
    for (int i = c.k - 1; i >= 0; i--) {
      // x = x * p_i + a_i (p_i applies for i < k - 1 only: start from a_{k-1})
      unsigned __int128 carry = a[i];
      if (i != c.k - 1) {
        const u64 p = c.p[i];
        for (int w = 0; w < n; w++) {
          const unsigned __int128 t = (unsigned __int128)x[w] * p + carry;
          x[w] = (u32)t;
          carry = t >> 32;
        }
      } else {
        n = 0;
      }
      while (carry) { x[n++] = (u32)carry; carry >>= 32; }
    }
    // symmetric representative: x > P / 2 -> x - P
    bool gt = false;  // 2x > P
    {
      int cmp = 0;
      u32 c2 = 0;
      u32 dbl[BW_PW + 1];
      for (int w = 0; w < BW_PW; w++) {
        dbl[w] = (x[w] << 1) | c2;
        c2 = x[w] >> 31;
      }
      dbl[BW_PW] = c2;
      for (int w = BW_PW; w >= 0 && !cmp; w--) {
        const u32 pv = w < c.pw ? c.P[w] : 0u;
        if (dbl[w] != pv) cmp = dbl[w] > pv ? 1 : -1;
      }
      gt = cmp > 0;
    }
    u32* dst = h + id * ow;
    if (gt) {  // x - P, two's complement over ow words
      u32 br = 0;
      for (int w = 0; w < ow; w++) {
        const u32 xv = w < BW_PW ? x[w] : 0u, pv = w < c.pw ? c.P[w] : 0u;
        const u64 t = (u64)xv - pv - br;
        dst[w] = (u32)t;
        br = (u32)(t >> 63);
      }
    } else {
      for (int w = 0; w < ow; w++) dst[w] = w < BW_PW ? x[w] : 0u;
    }
  }
}

__global__ void k_fold_err(const u32* src, u32* dst) {
  if (threadIdx.x == 0 && *src) atomicOr(dst, *src);
}

size_t al256w(size_t x) { return (x + 255) & ~(size_t)255; }

struct BwLayout { size_t off_rf, off_rg, off_out, off_mod, mod_bytes, total; int k; };

bool bw_layout(int variant, int batch, int lx, int ly, int cb, BwLayout& L) {
  L.k = nprimes(lx, ly, cb);
  if (L.k > BW_KMAX) return false;
  const size_t nin = (size_t)batch * lx * ly, nout = (size_t)batch * (2 * lx - 1) * (2 * ly - 1);
  size_t mod = 0;
  for (int i = 0; i < L.k; i++) {
    const size_t b = kmx_bks_mod_workspace_bytes(variant, batch, lx, ly, primes()[i]);
    if (!b) return false;
    mod = b > mod ? b : mod;
  }
  size_t o = 0;
  L.off_mod = o; L.mod_bytes = al256w(mod); o += L.mod_bytes;  // its error word leads (kmx_ws_status)
  L.off_rf = o; o += al256w((size_t)L.k * nin * 8);
  L.off_rg = o; o += al256w((size_t)L.k * nin * 8);
  L.off_out = o; o += al256w((size_t)L.k * nout * 8);
  L.total = o + 256;
  return true;
}

}  // namespace
}  // namespace kmx

using namespace kmx;

extern "C" {

int kmx_bks_wide_out_words(int lx, int ly, int coeff_bits) {
  if (lx < 1 || ly < 1 || coeff_bits < 1) return KMX_EINVAL;
  if (nprimes(lx, ly, coeff_bits) > BW_KMAX) return KMX_EINVAL;
  return (bound_bits(lx, ly, coeff_bits) + 1 + 31) / 32;  // + sign
}

size_t kmx_bks_wide_workspace_bytes(int variant, int batch, int lx, int ly, int coeff_bits) {
  if (variant < 1 || variant > 4 || batch < 0 || kmx_bks_wide_out_words(lx, ly, coeff_bits) < 0) return 0;
  BwLayout L;
  if (!bw_layout(variant, batch, lx, ly, coeff_bits, L)) return 0;
  return L.total;
}

int kmx_bks_wide_mul(int variant, int batch, int lx, int ly, int coeff_bits, const uint32_t* f, const uint32_t* g,
                     int in_words, uint32_t* h, int out_words, void* workspace, size_t ws_bytes, void* stream) {
  const int ow = kmx_bks_wide_out_words(lx, ly, coeff_bits);
  if (ow < 0 || variant < 1 || variant > 4 || batch < 0) return KMX_EINVAL;
  if (in_words < (coeff_bits + 1 + 31) / 32 || in_words > 64 || out_words < ow) return KMX_EINVAL;
  BwLayout L;
  if (!bw_layout(variant, batch, lx, ly, coeff_bits, L) || ws_bytes < L.total || !workspace) return KMX_EINVAL;
  g_launches = 0;
  if (batch == 0) return KMX_OK;
  CrtParams cp;
  if (!crt_params(L.k, cp)) return KMX_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  char* w = (char*)workspace;
  u32* err = (u32*)(w + L.off_mod);  // the first KS error word (kmx_ws_status reads offset 0)
  u32* err_in = (u32*)(w + L.total - 256);
  const long long nin = (long long)batch * lx * ly, nout = (long long)batch * (2 * lx - 1) * (2 * ly - 1);
  if (cudaMemsetAsync(err_in, 0, 4, st) != cudaSuccess) return KMX_ECUDA;
  u64* rf = (u64*)(w + L.off_rf);
  u64* rg = (u64*)(w + L.off_rg);
  u64* ro = (u64*)(w + L.off_out);
  const int grid_in = (int)((nin + 255) / 256 < 148 * 8 ? (nin + 255) / 256 : 148 * 8);
  k_wres<<<grid_in, 256, 0, st>>>(cp, f, nin, in_words, coeff_bits, rf, nin, err_in);
  k_wres<<<grid_in, 256, 0, st>>>(cp, g, nin, in_words, coeff_bits, rg, nin, err_in);
  if (cudaGetLastError() != cudaSuccess) return KMX_ECUDA;
  int nl = 2;
  for (int i = 0; i < L.k; i++) {
    const int rc = kmx_bks_mod_mul(variant, batch, lx, ly, cp.p[i], rf + i * nin, rg + i * nin, ro + i * nout,
                                   w + L.off_mod, L.mod_bytes, stream);
    if (rc) return rc;
    nl += kmx_last_launch_count();
    // each run clears the KS error word: keep its flags
    k_fold_err<<<1, 32, 0, st>>>(err, err_in);
    nl++;
  }
  const int grid_out = (int)((nout + 127) / 128 < 148 * 8 ? (nout + 127) / 128 : 148 * 8);
  k_garner<<<grid_out, 128, 0, st>>>(cp, ro, nout, nout, h, out_words);
  // every flag (input range, the k runs) into the word kmx_ws_status reads
  k_fold_err<<<1, 32, 0, st>>>(err_in, err);
  if (cudaGetLastError() != cudaSuccess) return KMX_ECUDA;
  g_launches = nl + 2;
  return KMX_OK;
}

int kmx_bks_wide_mul_host(int variant, int batch, int lx, int ly, int coeff_bits, const uint32_t* f,
                          const uint32_t* g, int in_words, uint32_t* h, int out_words) {
  struct Ctx {
    std::mutex mu;
    cudaStream_t st = nullptr;
    void* buf[3] = {nullptr, nullptr, nullptr};
    size_t cap[3] = {0, 0, 0};
  };
  static Ctx ctx[16];
  const size_t wsb = kmx_bks_wide_workspace_bytes(variant, batch, lx, ly, coeff_bits);
  if (!wsb) return KMX_EINVAL;
  if (batch == 0) return KMX_OK;
  const size_t fb = (size_t)batch * lx * ly * in_words * 4;
  const size_t hb = (size_t)batch * (2 * lx - 1) * (2 * ly - 1) * out_words * 4;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return KMX_ECUDA;
  Ctx& c = ctx[dev];
  std::lock_guard<std::mutex> lk(c.mu);
  if (!c.st && cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
  const size_t need[3] = {2 * al256w(fb), hb, wsb};
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
  u32* dF = (u32*)c.buf[0];
  u32* dG = (u32*)((char*)c.buf[0] + al256w(fb));
  if (cudaMemcpyAsync(dF, f, fb, cudaMemcpyHostToDevice, c.st) != cudaSuccess) return KMX_ECUDA;
  if (cudaMemcpyAsync(dG, g, fb, cudaMemcpyHostToDevice, c.st) != cudaSuccess) return KMX_ECUDA;
  int rc = kmx_bks_wide_mul(variant, batch, lx, ly, coeff_bits, dF, dG, in_words, (u32*)c.buf[1], out_words, c.buf[2],
                            c.cap[2], c.st);
  if (rc) return rc;
  if (cudaMemcpyAsync(h, c.buf[1], hb, cudaMemcpyDeviceToHost, c.st) != cudaSuccess) return KMX_ECUDA;
  return kmx_ws_status(c.buf[2], c.st);
}

}  // extern "C"
