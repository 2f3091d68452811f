// C ABI (include/kmx.h): parameter derivation, workspace planning and the
// per-variant launch sequence pack -> mul -> finish [-> recon] [-> bias].
//
// Variant sequences follow the reference exactly:
//   KS1 ksint.py:219-226   pack(N1) x2, one product, unpack out_len digits
//   KS2 ksint.py:229-247   pack/pack_reversed(N2), 2 products, out_len+1
//                          digits per stream, reversed list, reconstruction
//   KS3 ksint.py:257-279   pack/pack_negated(N2), 2 products, (P+-Q)/2,
//                          odd part >> N2, unpack at 2*N2, interleave
//   KS4 ksint.py:289-348   4 packs at N4, 4 products, even/odd half-sums,
//                          rev part >> N4 by parity of k, 2 reconstructions
//                          at 2*N4; KS1 fallback if not four_point_safe and
//                          the out_len == 1 single product (:299-303).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/kmx.h"
#include "kmx_common.cuh"
#include "kmx_internal.h"

using namespace kmx;

namespace {

int bitlen_u64(unsigned long long x) { return x ? 64 - __builtin_clzll(x) : 0; }
int getenv_int(const char* n, int d) {
  const char* v = getenv(n);
  return v && *v ? atoi(v) : d;
}
int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// K2 engine choice.  Default: the tcgen05 byte convolution wherever its shape
// gate admits the operands and the shorter one has more than 144 limbs; below
// that the integer-pipe schoolbook is faster (config-5 sweep with KMX_TC=0 vs
// default: the crossover sits at 134..145 limbs).  KMX_TC=0 forces the
// integer pipe, KMX_TC=1 the tensor cores wherever supported.
}  // namespace
namespace kmx {
// kmx_recon2.cu: in-place signed correction of coefficient records
cudaError_t launch_bias_apply(const BiasFix& bf, uint32_t* h, int out_words, int klen, long long h_pair_stride, int batch,
                              cudaStream_t st);

// chunked single-tile tensor-core multiply (kmx_tcj.cu)
bool tcj_plan(int ma, int mb, double* cost, bool short_only);
bool tc_plan_info(int ma, int mb, long long nprod, long long out[8]);
cudaError_t launch_tcmulj(const MulArgs& a, cudaStream_t st);
}  // namespace kmx
namespace {

// The chunked single-tile kernel (kmx_tcj.cu) for short products (plan with
// H0 <= 2, J >= 3) when the batch has too few products to fill the chip with
// the tiled kernel's CTAs (< 4 per SM): one CTA per product with a K span
// shortened by J is lower-latency there (c1 ks2/ks3 +9-11%, ks4 +8%), while
// the tiled kernel keeps the edge on full batches (c2 ks4 K2 0.121 vs 0.129 ms)
// and on long products (profiles/r01/tcj_sweep_*.json, c5 sweep).
// KMX_TCJ=1 / 0 forces it on / off wherever its shape gate admits the product.
bool use_tcj(int ma, int mb, long long nprod) {
  const char* v = getenv("KMX_TCJ");
  const int force = v && *v ? atoi(v) : -1;
  if (force == 0) return false;
  if (force < 0 && nprod >= 4LL * 148) return false;
  // the swizzled-window kernel (kmx_tcs.cu) beats it at c1 too (ks2 / ks3 K2
  // 16.8 -> 14.3 us, ks4 13.1 -> 12.8): chosen only where that kernel is off
  if (force < 0) {
    const char* ts = getenv("KMX_TCS");
    if (!(ts && *ts && atoi(ts) == 0)) return false;
  }
  return tcj_plan(ma, mb, nullptr, force < 0);
}

int tc_force() {  // read per call: tests switch KMX_TC inside one process
  const char* v = getenv("KMX_TC");
  return v && *v ? atoi(v) : -1;
}
bool use_tensor_mul(int ma, int mb) {
  const int force = tc_force();
  if (force == 0) return false;
  if (force < 0 && (ma < mb ? ma : mb) <= 144) return false;
  return tc_supported(ma, mb);
}
}  // namespace
namespace kmx {
bool mul_use_tensor(int ma, int mb) { return use_tensor_mul(ma, mb); }
// the product goes to one engine launch unless the tensor cores would be the
// engine of choice but cannot stage the operands (then Karatsuba splits it)
bool mul_engine_takes(int ma, int mb) {
  if (tc_force() == 0) return true;
  if (tc_force() < 0 && (ma < mb ? ma : mb) <= 144) return true;
  return tc_supported(ma, mb);
}
}  // namespace kmx
namespace {

// ---- tiny host bignum for the four-point bound (ksint.py:282-286)
typedef std::vector<uint32_t> Big;
Big big_from_u64(unsigned long long v) { Big r; while (v) { r.push_back((uint32_t)v); v >>= 32; } return r; }
Big big_pow2_minus1(int b) {  // 2^b - 1
  Big r((b + 31) / 32, 0xffffffffu);
  if (b % 32) r.back() = (1u << (b % 32)) - 1u;
  return r;
}
Big big_mul(const Big& a, const Big& b) {
  Big r(a.size() + b.size() + 1, 0u);
  for (size_t i = 0; i < a.size(); i++) {
    unsigned long long c = 0;
    for (size_t j = 0; j < b.size(); j++) {
      unsigned long long t = (unsigned long long)a[i] * b[j] + r[i + j] + c;
      r[i + j] = (uint32_t)t;
      c = t >> 32;
    }
    size_t k = i + b.size();
    while (c) { unsigned long long t = (unsigned long long)r[k] + c; r[k] = (uint32_t)t; c = t >> 32; k++; }
  }
  while (!r.empty() && r.back() == 0) r.pop_back();
  return r;
}
int big_cmp(Big a, Big b) {
  while (!a.empty() && a.back() == 0) a.pop_back();
  while (!b.empty() && b.back() == 0) b.pop_back();
  if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
  for (size_t i = a.size(); i-- > 0;) if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
  return 0;
}

struct KsPlan {
  int req_variant, variant, batch, lf, lg, b, in_words;
  unsigned flags;
  bool sign;
  int e, N1, N2, N4, out_len, out_words_min;
  bool safe;
  int N, P, kinds[4];
  int mf, mg, mp, mfs, mgs;
  int G, C, nbands, TI;
  long long ps;
  int ns;
  Stream st[4];
  int W, dwords, cnt_max, dslots;
  int nrs;
  ReconStream rs[2];
  size_t off_err, off_meta, off_opf, off_opg, off_prod, off_spill, off_dbuf, off_scr, off_cmap, off_kara, off_pseg,
      total;
  bool kara;
  bool wide;  // digits past the fast finish / reconstruction budgets (kmx_wide.cu)
  size_t off_wnum, off_wmaps, off_wscr;
  long long wt_stride;
  int fin_chunks;  // 256-limb chunks of the longest finish stream (chunk-parallel finish maps)
};

// words per digit-stream slot, rounded to 16 bytes (the pair reconstruction loads digit pairs)
static inline long long dslot_words(const KsPlan& p) { return ((long long)p.cnt_max * p.dwords + 3) & ~3LL; }

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// optional per-kernel CUDA-event timing of run_plan (kmx_prof_*):
// slots 0 pack, 1 mul, 2 finish, 3 recon, 4 bias
struct Prof {
  bool on = false;
  bool created = false;
  cudaEvent_t ev[6][2];
  bool used[6];
};
thread_local Prof g_prof;

void prof_begin(int slot, cudaStream_t st) {
  if (!g_prof.on) return;
  if (!g_prof.created) {
    for (int i = 0; i < 6; i++)
      for (int j = 0; j < 2; j++) cudaEventCreate(&g_prof.ev[i][j]);
    g_prof.created = true;
  }
  cudaEventRecord(g_prof.ev[slot][0], st);
  g_prof.used[slot] = true;
}
void prof_end(int slot, cudaStream_t st) {
  if (g_prof.on) cudaEventRecord(g_prof.ev[slot][1], st);
}
}  // namespace

namespace kmx {
void prof_mark(int slot, bool begin, cudaStream_t st) {
  if (begin) prof_begin(slot, st); else prof_end(slot, st);
}
bool prof_suspend() {
  const bool was = g_prof.on;
  g_prof.on = false;
  return was;
}
void prof_resume(bool was) { g_prof.on = was; }
void prof_reset() { for (int i = 0; i < 6; i++) g_prof.used[i] = false; }
void prof_keep(int slot) { g_prof.used[slot] = true; }
}  // namespace kmx

namespace {

int make_plan(KsPlan& p, int variant, int batch, int lf, int lg, int b, int in_words, unsigned flags) {
  memset(&p, 0, sizeof p);
  if (variant < 1 || variant > 4 || batch < 0 || lf < 1 || lg < 1 || b < 1) return KMX_EINVAL;
  p.req_variant = variant;
  p.batch = batch; p.lf = lf; p.lg = lg; p.b = b; p.flags = flags;
  p.sign = (flags & KMX_SIGNED) != 0;
  if (p.sign && b > 32) return KMX_EINVAL;
  if (in_words <= 0) in_words = (b + 31) / 32;
  if (p.sign && in_words != 1) return KMX_EINVAL;
  if (!p.sign && in_words < (b + 31) / 32) return KMX_EINVAL;
  p.in_words = in_words;
  // derive_params (ksint.py:82-98)
  p.e = bitlen_u64((unsigned long long)std::min(lf, lg) - 1);
  p.N1 = 2 * b + p.e;
  p.N2 = b + (p.e + 1) / 2;
  p.N4 = (p.N1 + 3) / 4;
  p.out_len = lf + lg - 1;
  p.out_words_min = (p.N1 + 31) / 32;
  // _four_point_safe (ksint.py:282-286): min(L)(2^b-1)^2 < 2^w (2^w - 1)
  {
    const int w = 2 * p.N4;
    Big t = big_pow2_minus1(b);
    Big lhs = big_mul(big_mul(t, t), big_from_u64((unsigned long long)std::min(lf, lg)));
    // rhs = 2^w (2^w - 1) = (2^w - 1) << w
    Big m1 = big_pow2_minus1(w);
    Big sh((size_t)(w / 32) + m1.size() + 1, 0u);
    for (size_t i = 0; i < m1.size(); i++) {
      unsigned long long v = (unsigned long long)m1[i] << (w % 32);
      sh[i + w / 32] |= (uint32_t)v;
      sh[i + w / 32 + 1] |= (uint32_t)(v >> 32);
    }
    p.safe = big_cmp(lhs, sh) < 0;
  }
  int v = variant;
  if (v == 4 && (!p.safe || p.out_len == 1)) v = 1;  // ksint.py:299-303
  p.variant = v;
  p.N = v == 1 ? p.N1 : (v == 4 ? p.N4 : p.N2);
  if (2 * p.N < b) return KMX_EINVAL;  // pack.py:55-59 (cannot happen for derived N)
  switch (v) {
    case 1: p.P = 1; p.kinds[0] = 0; break;
    case 2: p.P = 2; p.kinds[0] = 0; p.kinds[1] = 2; break;
    case 3: p.P = 2; p.kinds[0] = 0; p.kinds[1] = 1; break;
    default: p.P = 4; p.kinds[0] = 0; p.kinds[1] = 1; p.kinds[2] = 2; p.kinds[3] = 3; break;
  }
  // packed operand limbs: N (L-1) + b bits, +1 overlapped carry bit, +1 margin
  long long bf = (long long)p.N * (lf - 1) + b + 2;
  long long bg = (long long)p.N * (lg - 1) + b + 2;
  if ((bf + 31) / 32 > (1LL << 28) || (bg + 31) / 32 > (1LL << 28)) return KMX_EINVAL;
  p.mf = (int)((bf + 31) / 32);
  p.mg = (int)((bg + 31) / 32);
  p.mfs = (p.mf + 3) & ~3;
  p.mgs = (p.mg + 3) & ~3;
  p.mp = p.mf + p.mg;
  // multiply geometry (kmx_mul.cu): G = row split, C = band columns
  mul_geometry(p.mf, p.mg, &p.G, &p.C, &p.nbands, &p.TI);
  p.ps = (long long)p.nbands * p.C;
  // output streams (finish) and reconstructions
  const int k = p.out_len, n_even = (k + 1) / 2, n_odd = k / 2;
  auto S = [&](int i) -> Stream& { return p.st[i]; };
  memset(p.st, 0, sizeof p.st);
  p.nrs = 0;
  if (v == 1) {
    p.ns = 1; p.W = p.N1;
    S(0) = Stream{0, 0, 0, 0, 0, p.N1, k, 0, 0, 1, 0, 0};
  } else if (v == 2) {
    p.ns = 2; p.W = p.N2;
    S(0) = Stream{0, 0, 0, 0, 0, p.N2, k + 1, 1, 0, 0, 0, 0};
    S(1) = Stream{1, 0, 0, 0, 0, p.N2, k + 1, 1, 0, 0, 1, 1};
    p.nrs = 1;
    p.rs[0] = ReconStream{0, 1, k, 0, 1};
    p.cnt_max = k + 1; p.dslots = 2;
  } else if (v == 3) {
    p.ns = 2; p.W = 2 * p.N2;
    S(0) = Stream{0, 1, +1, 1, 1, 2 * p.N2, n_even, 0, 0, 2, 0, 0};
    S(1) = Stream{0, 1, -1, 1, 1 + p.N2, 2 * p.N2, n_odd, 0, 1, 2, 0, 0};
  } else {
    const int w = 2 * p.N4;
    p.ns = 4; p.W = w;
    S(0) = Stream{0, 1, +1, 1, 1, w, n_even + 1, 1, 0, 0, 0, 0};
    S(1) = Stream{0, 1, -1, 1, 1 + p.N4, w, n_odd + 1, 1, 0, 0, 1, 0};
    S(2) = Stream{2, 3, +1, 3, 1 + (k % 2 == 0 ? p.N4 : 0), w, n_even + 1, 1, 0, 0, 2, 1};
    S(3) = Stream{2, 3, -1, 3, 1 + (k % 2 == 1 ? p.N4 : 0), w, n_odd + 1, 1, 0, 0, 3, 1};
    p.nrs = n_odd ? 2 : 1;
    p.rs[0] = ReconStream{0, 2, n_even, 0, 2};
    p.rs[1] = ReconStream{1, 3, n_odd, 1, 2};
    p.cnt_max = n_even + 1; p.dslots = 4;
  }
  p.dwords = (p.W + 31) / 32;
  p.wide = p.W > 32 * (FIN_HALO - 1) || (p.nrs && p.dwords > 17) || (getenv_int("KMX_WIDE", 0) == 1 && !p.sign);
  if (p.wide && p.sign) return KMX_EINVAL;  // signed inputs have b <= 32: never wide
  // workspace layout
  size_t o = 0;
  p.off_err = o; o = align256(o + 16);
  p.off_meta = o; o = align256(o + (size_t)batch * p.P * 2 * 2 * 4);
  p.off_opf = o; o = align256(o + (size_t)batch * p.P * p.mfs * 4);
  p.off_opg = o; o = align256(o + (size_t)batch * p.P * p.mgs * 4);
  p.off_prod = o; o = align256(o + (size_t)batch * p.P * p.ps * 4);
  p.off_spill = o; o = align256(o + (size_t)batch * p.P * p.nbands * 16);
  p.off_dbuf = o;
  if (p.nrs) o = align256(o + (size_t)batch * p.dslots * dslot_words(p) * 4);
  p.off_scr = o;
  if (p.sign) o = align256(o + (size_t)batch * (lf + lg + 2) * 8);
  {  // chunk-parallel finish: one carry-map byte per (stream, 256-limb chunk)
    long long qd = 0;
    for (int i = 0; i < p.ns; i++) {
      const long long E = p.st[i].off + (long long)p.st[i].cnt * p.st[i].W;
      long long q = p.mp + 1;
      if ((E + 31) / 32 + 1 > q) q = (E + 31) / 32 + 1;
      if (q > qd) qd = q;
    }
    p.fin_chunks = (int)((qd + 255) / 256);
  }
  p.off_cmap = o;
  o = align256(o + (size_t)batch * p.ns * p.fin_chunks);
  // segmented pack scratch (kmx_packseg.cu)
  p.off_pseg = o;
  o = align256(o + pack_seg_scratch_bytes(batch, 2 * p.P, std::max(p.mf, p.mg)));
  // Karatsuba levels above the engines (kmx_kara.cu): sums, sub-products, maps
  p.kara = kara_used(p.mf, p.mg);
  p.off_kara = o;
  if (p.kara) o = align256(o + kara_ws_bytes(p.mf, p.mg, (long long)batch * p.P));
  if (p.wide) {  // normalized stream numerators, their carry maps, reconstruction scratch
    p.wt_stride = (p.mp + 1 + 3) & ~3LL;
    p.off_wnum = o; o = align256(o + (size_t)batch * p.wt_stride * 4);
    p.off_wmaps = o; o = align256(o + lc_map_bytes(batch, p.mp + 1));
    p.off_wscr = o; o = align256(o + wide_recon_scratch_words(batch, p.nrs, p.dwords) * 4);
  }
  p.total = o;
  return KMX_OK;
}

int cuda_rc(cudaError_t e) { return e == cudaSuccess ? KMX_OK : KMX_ECUDA; }

// finish + reconstruction for wide digits (kmx_wide.cu): per stream, the
// numerator P +- sgn(Q)|Q| normalized by the linear-combination kernels, a
// bit-field gather of its digits, then the multiword reconstruction
int run_wide(const KsPlan& p, const FinishArgs& fa, char* w, cudaStream_t st) {
  uint32_t* T = (uint32_t*)(w + p.off_wnum);
  cudaError_t e;
  for (int i = 0; i < p.ns; i++) {
    const Stream& S = p.st[i];
    LcArgs la;
    memset(&la, 0, sizeof la);
    la.maps = w + p.off_wmaps;
    la.err = fa.err;
    la.nt = 1;
    const long long pstr = (long long)p.P * p.ps, sstr = (long long)p.P * p.nbands * 2;
    la.t[0] = LcTerm{fa.P + (long long)S.zP * p.ps, pstr, p.mp, 0, +1, fa.spill + (long long)S.zP * p.nbands * 2,
                     p.nbands, sstr, nullptr, 0, 0};
    if (S.qsign) {
      la.nt = 2;
      la.t[1] = LcTerm{fa.P + (long long)S.zQ * p.ps, pstr, p.mp, 0, S.qsign, fa.spill + (long long)S.zQ * p.nbands * 2,
                       p.nbands, sstr, fa.meta + 2 * S.qmeta, fa.meta_per_pair, 2 * fa.mf_slot_stride};
    }
    la.out = T;
    la.out_stride = p.wt_stride;
    la.out_len = p.mp + 1;
    if ((e = launch_lincomb(la, p.batch, st)) != cudaSuccess) return KMX_ECUDA;
    WideDigitArgs wa;
    memset(&wa, 0, sizeof wa);
    wa.T = T; wa.t_stride = p.wt_stride; wa.t_len = p.mp + 1;
    wa.s = S;
    wa.h = fa.h; wa.out_words = fa.out_words; wa.h_pair_stride = fa.h_pair_stride;
    wa.dbuf = fa.dbuf; wa.dwords = fa.dwords; wa.dslot_stride = fa.dslot_stride; wa.dslots_pair = fa.dslots_pair;
    wa.err = fa.err;
    wa.batch = p.batch;
    if ((e = launch_wide_digits(wa, st)) != cudaSuccess) return KMX_ECUDA;
    g_launches += 3;
  }
  if (p.nrs) {
    ReconArgs ra;
    memset(&ra, 0, sizeof ra);
    for (int i = 0; i < p.nrs; i++) ra.s[i] = p.rs[i];
    ra.ns = p.nrs; ra.batch = p.batch; ra.W = p.W;
    ra.dbuf = fa.dbuf; ra.dwords = p.dwords; ra.dslot_stride = fa.dslot_stride; ra.dslots_pair = p.dslots;
    ra.h = fa.h; ra.out_words = fa.out_words; ra.h_pair_stride = fa.h_pair_stride;
    ra.err = fa.err;
    if ((e = launch_wide_recon(ra, (uint32_t*)(w + p.off_wscr), st)) != cudaSuccess) return KMX_ECUDA;
    g_launches++;
  }
  return KMX_OK;
}

int run_plan(const KsPlan& p, const uint32_t* f, const uint32_t* g, uint32_t* h, int out_words,
             void* ws, size_t ws_bytes, cudaStream_t st, uint32_t* err_shared = nullptr,
             cudaEvent_t after_pack = nullptr) {
  g_launches = 0;
  if (out_words < p.out_words_min) return KMX_EINVAL;
  if (ws_bytes < p.total || (!ws && p.total)) return KMX_EINVAL;
  if (p.batch == 0) return KMX_OK;
  for (int i = 0; i < 6; i++) g_prof.used[i] = false;
  char* w = (char*)ws;
  uint32_t* err = (uint32_t*)(w + p.off_err);
  uint32_t* meta = (uint32_t*)(w + p.off_meta);
  uint32_t* opf = (uint32_t*)(w + p.off_opf);
  uint32_t* opg = (uint32_t*)(w + p.off_opg);
  uint32_t* prod = (uint32_t*)(w + p.off_prod);
  unsigned long long* spill = (unsigned long long*)(w + p.off_spill);
  uint32_t* dbuf = (uint32_t*)(w + p.off_dbuf);
  unsigned long long* scr = (unsigned long long*)(w + p.off_scr);
  cudaError_t e = cudaMemsetAsync(err, 0, 12, st);  // error flag, multiply work counter, recon fallbacks
  if (e != cudaSuccess) return KMX_ECUDA;
  uint32_t* const cnt = err + 1;  // multiply work counter
  uint32_t* const diag = err + 2;
  if (err_shared) err = err_shared;  // split batch: both halves latch into one flag

  PackArgs pa;
  memset(&pa, 0, sizeof pa);
  pa.nops = 2 * p.P;
  pa.N = p.N; pa.b = p.b; pa.in_words = p.in_words; pa.bias = p.sign; pa.err = err;
  pa.scratch = w + p.off_pseg;
  pa.scratch_bytes = pack_seg_scratch_bytes(p.batch, 2 * p.P, std::max(p.mf, p.mg));
  const bool validate = !(p.flags & KMX_NO_VALIDATE);
  for (int s = 0; s < p.P; s++) {
    PackOp& F = pa.op[s];
    F.coeffs = f; F.coeff_pair_stride = (long long)p.lf * p.in_words; F.len = p.lf; F.kind = p.kinds[s];
    F.out = opf + (long long)s * p.mfs; F.out_pair_stride = (long long)p.P * p.mfs;
    F.meta = meta + 2 * s; F.meta_pair_stride = 4LL * p.P; F.m = p.mf; F.validate = validate && s == 0;
    PackOp& Gq = pa.op[p.P + s];
    Gq.coeffs = g; Gq.coeff_pair_stride = (long long)p.lg * p.in_words; Gq.len = p.lg; Gq.kind = p.kinds[s];
    Gq.out = opg + (long long)s * p.mgs; Gq.out_pair_stride = (long long)p.P * p.mgs;
    Gq.meta = meta + 2 * (p.P + s); Gq.meta_pair_stride = 4LL * p.P; Gq.m = p.mg; Gq.validate = validate && s == 0;
    if (p.sign && s == 0) {  // prefix sums of the lifted inputs for the fused bias correction
      F.prefix = scr; F.prefix_pair_stride = p.lf + p.lg + 2;
      Gq.prefix = scr + p.lf + 1; Gq.prefix_pair_stride = p.lf + p.lg + 2;
    }
  }
  BiasFix bfix;
  memset(&bfix, 0, sizeof bfix);
  if (p.sign) {
    bfix.pf = scr; bfix.pair_stride = p.lf + p.lg + 2;
    bfix.lf = p.lf; bfix.lg = p.lg; bfix.b = p.b; bfix.enabled = 1; bfix.lgpad = -1;
  }
  // K2 engine; with the tensor cores K1 can be fused into K2's prologue when
  // the coefficient vectors can be staged in shared memory (KMX_FUSE=1).  Off
  // by default: with one-shot CTAs the pack latency is exposed in front of
  // the MMAs (c2 ks4: 0.27 ms fused vs 0.08 + 0.12 ms separate).
  const bool tc = !p.kara && use_tensor_mul(p.mf, p.mg);
  int lmax = p.lf > p.lg ? p.lf : p.lg;
  const size_t stage = (size_t)(lmax + PK_PAD_WORDS) * p.in_words * 4;
  const char* fz = getenv("KMX_FUSE");
  const bool fuse = tc && (fz && *fz && atoi(fz) == 1) &&
                    (size_t)(lmax + PK_PAD_WORDS) * p.in_words <= (size_t)PK_STAGE_LIMIT_WORDS &&
                    tc_supported(p.mf, p.mg, stage);
  if (!fuse) {
    prof_begin(0, st);
    if ((e = launch_pack(pa, p.batch, st)) != cudaSuccess) return KMX_ECUDA;
    prof_end(0, st);
    g_launches++;
  }
  if (after_pack && cudaEventRecord(after_pack, st) != cudaSuccess) return KMX_ECUDA;

  MulArgs ma;
  memset(&ma, 0, sizeof ma);
  ma.flags_no_tune = (p.flags & KMX_NO_TUNE) != 0;
  ma.A = opf; ma.a_stride = p.mfs; ma.ma = p.mf;
  ma.B = opg; ma.b_stride = p.mgs; ma.mb = p.mg;
  ma.P = prod; ma.p_stride = p.ps; ma.spill = spill;
  ma.nprod = p.batch * p.P; ma.nbands = p.nbands; ma.G = p.G; ma.TI = p.TI;
  ma.counter = (int*)cnt;
  ma.err = err;
  FinishArgs fa;
  memset(&fa, 0, sizeof fa);
  for (int i = 0; i < p.ns; i++) fa.s[i] = p.st[i];
  fa.ns = p.ns;
  fa.P = prod; fa.p_stride = p.ps; fa.mp = p.mp; fa.nprod_pair = p.P;
  fa.spill = spill; fa.nbands = p.nbands; fa.band_cols = p.C;
  fa.meta = meta; fa.meta_per_pair = 4 * p.P; fa.mf_slot_stride = p.P;
  fa.h = h; fa.out_words = out_words; fa.h_pair_stride = (long long)p.out_len * out_words;
  fa.dbuf = dbuf; fa.dwords = p.dwords; fa.dslot_stride = dslot_words(p);
  fa.dslots_pair = p.dslots; fa.err = err;
  fa.bias = bfix;
  fa.cmaps = (uint8_t*)(w + p.off_cmap);
  fa.nchunks = p.fin_chunks;
  // ks1 / ks3 with signed inputs: the finish writes the lifted product's coefficients and a
  // streaming pass corrects them in place (kmx_recon2.cu; KMX_BIAS_FUSED=1: inside the finish)
  static const int bias_fused = getenv_int("KMX_BIAS_FUSED", 0);
  const bool bias_pass = p.sign && !p.nrs && !bias_fused && p.batch <= 65535;
  if (bias_pass) fa.bias.enabled = 0;
  bool finished = false;  // K3 already ran inside K2
  prof_begin(1, st);
  if (p.kara) {
    int nl = 0;
    if ((e = launch_kara(ma, w + p.off_kara, st, &nl)) != cudaSuccess) return KMX_ECUDA;
    g_launches += nl - 1;
  } else if (tc && !fuse && use_tcj(p.mf, p.mg, (long long)p.batch * p.P)) {
    if ((e = launch_tcmulj(ma, st)) != cudaSuccess) return KMX_ECUDA;
  } else if (tc) {
    // single-tile products with a warp-per-stream K3: K2 + K3 in one kernel
    if (!fuse && !p.wide && launch_tcmul_finish(ma, fa, p.batch, st, &e)) {
      if (e != cudaSuccess) return KMX_ECUDA;
      finished = true;
    } else if ((e = launch_tcmul(ma, st, fuse ? &pa : nullptr, p.P)) != cudaSuccess) return KMX_ECUDA;
  } else {
    if ((e = launch_mul(ma, st)) != cudaSuccess) return KMX_ECUDA;
  }
  prof_end(1, st);
  g_launches++;

  ReconArgs ra;
  memset(&ra, 0, sizeof ra);
  if (p.wide) return run_wide(p, fa, w, st);
  if (p.nrs) {
    for (int i = 0; i < p.nrs; i++) ra.s[i] = p.rs[i];
    ra.ns = p.nrs; ra.batch = p.batch; ra.W = p.W;
    ra.dbuf = dbuf; ra.dwords = p.dwords; ra.dslot_stride = dslot_words(p);
    ra.dslots_pair = p.dslots;
    ra.h = h; ra.out_words = out_words; ra.h_pair_stride = (long long)p.out_len * out_words;
    ra.err = err;
    ra.bias = bfix;
    ra.diag = diag;
    // ks2 / ks4: finish + reconstruct in one kernel (k_finrec) when both fit it
    bool fused = false;
    prof_begin(3, st);
    if (!finished && (e = launch_finrec(fa, ra, p.batch, st, &fused)) != cudaSuccess) return KMX_ECUDA;
    if (fused) {
      prof_end(3, st);
      g_launches++;
      return KMX_OK;
    }
  }
  if (!finished) {
    prof_begin(2, st);
    if ((e = launch_finish(fa, p.batch, st)) != cudaSuccess) return KMX_ECUDA;
    prof_end(2, st);
    g_launches++;
  }
  if (bias_pass) {
    prof_begin(4, st);
    if ((e = launch_bias_apply(bfix, h, out_words, p.out_len, (long long)p.out_len * out_words, p.batch, st)) !=
        cudaSuccess)
      return KMX_ECUDA;
    prof_end(4, st);
    g_launches++;
  }

  if (p.nrs) {
    prof_begin(3, st);
    if ((e = launch_recon(ra, st)) != cudaSuccess) return KMX_ECUDA;
    prof_end(3, st);
    g_launches++;
  }
  return KMX_OK;
}

int status_from_flag(uint32_t fl) {
  if (fl & ERR_INVAL) return KMX_EINVAL;
  if (fl & ERR_RECON) return KMX_ERECON;
  if (fl & ERR_INEXACT) return KMX_EINEXACT;
  return KMX_OK;
}

// per-device cached buffers for the host entry points
constexpr int HOST_LANES = 3;     // streams of the pipelined host path
constexpr int HOST_MAX_CHUNKS = 16;

struct HostLane {
  cudaStream_t st = nullptr;
  void* buf[3] = {nullptr, nullptr, nullptr};
  size_t cap[3] = {0, 0, 0};
};

struct HostCtx {
  std::mutex mu;
  cudaStream_t st = nullptr;
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t cap[4] = {0, 0, 0, 0};
  HostLane lane[HOST_LANES];
  uint32_t* flags = nullptr;        // pinned, one error word per chunk
  // copy-engine pipeline (ks_mul_host_streams): one H2D stream, two compute
  // streams, one D2H stream; whole-batch device buffers
  cudaStream_t s_in = nullptr, s_out = nullptr, s_comp[2] = {nullptr, nullptr};
  cudaEvent_t ev_in[HOST_MAX_CHUNKS] = {}, ev_done[HOST_MAX_CHUNKS] = {};
  void* pbuf[4] = {nullptr, nullptr, nullptr, nullptr};  // f+g, h, ws0, ws1
  size_t pcap[4] = {0, 0, 0, 0};
};

int ensure_buf(void** buf, size_t* cap, size_t bytes) {
  if (*cap >= bytes) return KMX_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *cap = 0;
  size_t want = std::max(bytes, (size_t)4096);
  if (cudaMalloc(buf, want) != cudaSuccess) return KMX_ENOMEM;
  *cap = want;
  return KMX_OK;
}
HostCtx g_ctx[16];

int ensure(HostCtx& c, int i, size_t bytes) {
  if (c.cap[i] >= bytes) return KMX_OK;
  if (c.buf[i]) cudaFree(c.buf[i]);
  c.buf[i] = nullptr;
  c.cap[i] = 0;
  size_t want = std::max(bytes, (size_t)4096);
  if (cudaMalloc(&c.buf[i], want) != cudaSuccess) return KMX_ENOMEM;
  c.cap[i] = want;
  return KMX_OK;
}

HostCtx* host_ctx(int* rc) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) { *rc = KMX_ECUDA; return nullptr; }
  HostCtx& c = g_ctx[dev];
  *rc = KMX_OK;
  return &c;
}

// Pipelined host path: the batch is cut into chunks that rotate over
// HOST_LANES streams, so the host->device copy of chunk i+1, the kernels of
// chunk i and the device->host copy of chunk i-1 overlap (with pinned host
// buffers; pageable buffers still work, without the overlap).
int ks_mul_host_pipelined(const KsPlan& pfull, HostCtx* c, const uint32_t* f, const uint32_t* g,
                                 uint32_t* h, int out_words, int nchunks) {
  const int batch = pfull.batch;
  const int cb = (batch + nchunks - 1) / nchunks;
  nchunks = (batch + cb - 1) / cb;
  KsPlan pc, pt;
  int rc = make_plan(pc, pfull.req_variant, cb, pfull.lf, pfull.lg, pfull.b, pfull.in_words, pfull.flags);
  if (rc) return rc;
  const int tail = batch - (nchunks - 1) * cb;
  rc = make_plan(pt, pfull.req_variant, tail, pfull.lf, pfull.lg, pfull.b, pfull.in_words, pfull.flags);
  if (rc) return rc;
  const size_t fpp = (size_t)pfull.lf * pfull.in_words, gpp = (size_t)pfull.lg * pfull.in_words;
  const size_t hpp = (size_t)pfull.out_len * out_words;
  const size_t fb = (size_t)cb * fpp * 4, gb = (size_t)cb * gpp * 4, hb = (size_t)cb * hpp * 4;
  if (!c->flags && cudaMallocHost(&c->flags, HOST_MAX_CHUNKS * sizeof(uint32_t)) != cudaSuccess) return KMX_ENOMEM;
  for (int l = 0; l < HOST_LANES && l < nchunks; l++) {
    HostLane& L = c->lane[l];
    if (!L.st && cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
    if ((rc = ensure_buf(&L.buf[0], &L.cap[0], align256(fb) + gb + 256))) return rc;
    if ((rc = ensure_buf(&L.buf[1], &L.cap[1], hb))) return rc;
    if ((rc = ensure_buf(&L.buf[2], &L.cap[2], pc.total))) return rc;
  }
  int nl = 0;
  for (int i = 0; i < nchunks; i++) {
    HostLane& L = c->lane[i % HOST_LANES];
    const KsPlan& pp = (i == nchunks - 1) ? pt : pc;
    const int bi = pp.batch;
    uint32_t* df = (uint32_t*)L.buf[0];
    uint32_t* dg = (uint32_t*)((char*)L.buf[0] + align256(fb));
    if (cudaMemcpyAsync(df, f + (size_t)i * cb * fpp, (size_t)bi * fpp * 4, cudaMemcpyHostToDevice, L.st) != cudaSuccess)
      return KMX_ECUDA;
    if (cudaMemcpyAsync(dg, g + (size_t)i * cb * gpp, (size_t)bi * gpp * 4, cudaMemcpyHostToDevice, L.st) != cudaSuccess)
      return KMX_ECUDA;
    rc = run_plan(pp, df, dg, (uint32_t*)L.buf[1], out_words, L.buf[2], L.cap[2], L.st);
    if (rc) return rc;
    nl += g_launches;
    if (cudaMemcpyAsync(h + (size_t)i * cb * hpp, L.buf[1], (size_t)bi * hpp * 4, cudaMemcpyDeviceToHost, L.st) != cudaSuccess)
      return KMX_ECUDA;
    if (cudaMemcpyAsync(c->flags + i, L.buf[2], 4, cudaMemcpyDeviceToHost, L.st) != cudaSuccess) return KMX_ECUDA;
  }
  for (int l = 0; l < HOST_LANES && l < nchunks; l++)
    if (cudaStreamSynchronize(c->lane[l].st) != cudaSuccess) return KMX_ECUDA;
  g_launches = nl;
  uint32_t fl = 0;
  for (int i = 0; i < nchunks; i++) fl |= c->flags[i];
  return status_from_flag(fl);
}

// Copy-engine pipeline: every chunk's host->device copy is queued on one
// stream (back to back at full link speed), its kernels on one of two compute
// streams (waiting on that copy's event; the two streams overlap one chunk's
// latency-bound stages with the next one's), and its device->host copy on a
// fourth stream (waiting on the kernels' event), so the device->host direction
// -- 3x the bytes of the other at c2 -- streams continuously once the first
// chunk is done.  KMX_HOST_PIPE=0 selects the lane pipeline above.
int ks_mul_host_streams(const KsPlan& pfull, HostCtx* c, const uint32_t* f, const uint32_t* g, uint32_t* h,
                        int out_words, int nchunks) {
  const auto t_start = std::chrono::steady_clock::now();
  const int batch = pfull.batch;
  // Equal chunks; KMX_HOST_GEOM=1 tries geometric ones (a small first chunk
  // starts the device->host stream early, later chunks double): measured
  // 0.748 vs 0.718 ms per c2 step, so off by default.
  static const int geom = getenv("KMX_HOST_GEOM") ? atoi(getenv("KMX_HOST_GEOM")) : 0;
  int starts[HOST_MAX_CHUNKS + 1];
  int nch = 0;
  if (geom) {
    int sz = std::max(1, batch / 16), o = 0;
    while (o < batch && nch < HOST_MAX_CHUNKS) {
      int take = (nch == HOST_MAX_CHUNKS - 1 || o + sz >= batch || o + 2 * sz > batch) ? batch - o : sz;
      starts[nch++] = o;
      o += take;
      sz *= 2;
    }
    starts[nch] = batch;
  } else {
    const int cb = (batch + nchunks - 1) / nchunks;
    for (int o = 0; o < batch; o += cb) starts[nch++] = o;
    starts[nch] = batch;
  }
  nchunks = nch;
  KsPlan plans[HOST_MAX_CHUNKS];
  size_t ws_need = 0;
  for (int i = 0; i < nchunks; i++) {
    const int rc = make_plan(plans[i], pfull.req_variant, starts[i + 1] - starts[i], pfull.lf, pfull.lg, pfull.b,
                             pfull.in_words, pfull.flags);
    if (rc) return rc;
    ws_need = std::max(ws_need, plans[i].total);
  }
  int rc;
  const size_t fpp = (size_t)pfull.lf * pfull.in_words, gpp = (size_t)pfull.lg * pfull.in_words;
  const size_t hpp = (size_t)pfull.out_len * out_words;
  const size_t fb = (size_t)batch * fpp * 4, gb = (size_t)batch * gpp * 4, hb = (size_t)batch * hpp * 4;
  if (!c->flags && cudaMallocHost(&c->flags, HOST_MAX_CHUNKS * sizeof(uint32_t)) != cudaSuccess) return KMX_ENOMEM;
  auto mk = [](cudaStream_t* s) { return *s || cudaStreamCreateWithFlags(s, cudaStreamNonBlocking) == cudaSuccess; };
  if (!mk(&c->s_in) || !mk(&c->s_out) || !mk(&c->s_comp[0]) || !mk(&c->s_comp[1])) return KMX_ECUDA;
  for (int i = 0; i < nchunks; i++) {
    if (!c->ev_in[i] && cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming) != cudaSuccess) return KMX_ECUDA;
    if (!c->ev_done[i] && cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming) != cudaSuccess)
      return KMX_ECUDA;
  }
  if ((rc = ensure_buf(&c->pbuf[0], &c->pcap[0], align256(fb) + gb + 256))) return rc;
  if ((rc = ensure_buf(&c->pbuf[1], &c->pcap[1], hb))) return rc;
  if ((rc = ensure_buf(&c->pbuf[2], &c->pcap[2], ws_need))) return rc;
  if ((rc = ensure_buf(&c->pbuf[3], &c->pcap[3], ws_need))) return rc;
  uint32_t* df = (uint32_t*)c->pbuf[0];
  uint32_t* dg = (uint32_t*)((char*)c->pbuf[0] + align256(fb));
  uint32_t* dh = (uint32_t*)c->pbuf[1];
  int nl = 0;
  static const int tr = getenv("KMX_HOST_TRACE") ? atoi(getenv("KMX_HOST_TRACE")) : 0;
  cudaEvent_t tev[3 * HOST_MAX_CHUNKS + 1];
  if (tr >= 2) {
    for (int i = 0; i < 3 * nchunks + 1; i++) cudaEventCreate(&tev[i]);
    cudaEventRecord(tev[3 * nchunks], c->s_in);
  }
  for (int i = 0; i < nchunks; i++) {
    const KsPlan& pp = plans[i];
    const size_t o = (size_t)starts[i];
    const int bi = pp.batch;
    if (cudaMemcpyAsync(df + o * fpp, f + o * fpp, (size_t)bi * fpp * 4, cudaMemcpyHostToDevice, c->s_in) != cudaSuccess ||
        cudaMemcpyAsync(dg + o * gpp, g + o * gpp, (size_t)bi * gpp * 4, cudaMemcpyHostToDevice, c->s_in) != cudaSuccess ||
        cudaEventRecord(c->ev_in[i], c->s_in) != cudaSuccess)
      return KMX_ECUDA;
    if (tr >= 2) cudaEventRecord(tev[3 * i], c->s_in);
    static const int ncs = getenv("KMX_HOST_COMP_STREAMS") ? atoi(getenv("KMX_HOST_COMP_STREAMS")) : 2;
    const int cs = ncs >= 2 ? (i & 1) : 0;
    cudaStream_t sc = c->s_comp[cs];
    if (cudaStreamWaitEvent(sc, c->ev_in[i], 0) != cudaSuccess) return KMX_ECUDA;
    void* ws = c->pbuf[2 + cs];
    rc = run_plan(pp, df + o * fpp, dg + o * gpp, dh + o * hpp, out_words, ws, c->pcap[2 + cs], sc);
    if (rc) return rc;
    nl += g_launches;
    if (cudaMemcpyAsync(c->flags + i, ws, 4, cudaMemcpyDeviceToHost, sc) != cudaSuccess ||
        cudaEventRecord(c->ev_done[i], sc) != cudaSuccess)
      return KMX_ECUDA;
    if (tr >= 2) cudaEventRecord(tev[3 * i + 1], sc);
    if (cudaStreamWaitEvent(c->s_out, c->ev_done[i], 0) != cudaSuccess ||
        cudaMemcpyAsync(h + o * hpp, dh + o * hpp, (size_t)bi * hpp * 4, cudaMemcpyDeviceToHost, c->s_out) != cudaSuccess)
      return KMX_ECUDA;
    if (tr >= 2) cudaEventRecord(tev[3 * i + 2], c->s_out);
  }
  static const int trace = getenv("KMX_HOST_TRACE") ? atoi(getenv("KMX_HOST_TRACE")) : 0;
  const auto t_enq = std::chrono::steady_clock::now();
  if (cudaStreamSynchronize(c->s_out) != cudaSuccess || cudaStreamSynchronize(c->s_comp[0]) != cudaSuccess ||
      cudaStreamSynchronize(c->s_comp[1]) != cudaSuccess)
    return KMX_ECUDA;
  if (tr >= 2) {
    for (int i = 0; i < nchunks; i++) {
      float a = 0, b = 0, d = 0;
      cudaEventElapsedTime(&a, tev[3 * nchunks], tev[3 * i]);
      cudaEventElapsedTime(&b, tev[3 * nchunks], tev[3 * i + 1]);
      cudaEventElapsedTime(&d, tev[3 * nchunks], tev[3 * i + 2]);
      fprintf(stderr, "  chunk %d (%d pairs): h2d done %.1f us, kernels done %.1f us, d2h done %.1f us\n", i,
              plans[i].batch, 1e3 * a, 1e3 * b, 1e3 * d);
    }
    for (int i = 0; i < 3 * nchunks + 1; i++) cudaEventDestroy(tev[i]);
  }
  if (trace) {
    const auto t_end = std::chrono::steady_clock::now();
    fprintf(stderr, "kmx host: %d chunks, enqueue %.1f us, enqueue-to-done %.1f us\n", nchunks,
            std::chrono::duration<double, std::micro>(t_enq - t_start).count(),
            std::chrono::duration<double, std::micro>(t_end - t_enq).count());
  }
  g_launches = nl;
  uint32_t fl = 0;
  for (int i = 0; i < nchunks; i++) fl |= c->flags[i];
  return status_from_flag(fl);
}

// Split a device batch into K parts on K streams (kmx_ks_mul; K = 2 by
// default, KMX_SPLIT_WAYS up to 4) for batches >= 256 pairs; KMX_SPLIT=0/1
// forces, the KMX_NO_SPLIT flag disables per call.  The workspace is always
// sized for the split; the call runs unsplit while per-kernel profiling is on
// (kmx_prof_*).
constexpr int SPLIT_MAX = 4;
// A schedule: the batch cut into `ways` parts on `ways` streams, all started
// at the fork or (stagger) each when the previous part's pack is done.
struct Sched { int ways, stagger; };
constexpr Sched SCHEDS[] = {{1, 0}, {2, 0}, {2, 1}, {4, 1}};
constexpr int NSCHED = 4;

// Default (no measurement): two parts at >= 256 pairs.  KMX_SPLIT=0 forces one
// part, KMX_SPLIT=1 the default split with KMX_SPLIT_WAYS / KMX_SPLIT_STAGGER.
int split_force() {
  static const int f = getenv("KMX_SPLIT") ? atoi(getenv("KMX_SPLIT")) : -1;
  return f;
}
Sched default_sched(int batch, unsigned flags) {
  static const int ways = getenv("KMX_SPLIT_WAYS") ? atoi(getenv("KMX_SPLIT_WAYS")) : 2;
  static const int stag = getenv("KMX_SPLIT_STAGGER") ? atoi(getenv("KMX_SPLIT_STAGGER")) : 0;
  if ((flags & KMX_NO_SPLIT) || split_force() == 0) return Sched{1, 0};
  if (!(split_force() == 1 || batch >= 256)) return Sched{1, 0};
  int k = ways < 2 ? 2 : (ways > SPLIT_MAX ? SPLIT_MAX : ways);
  if (k > batch) k = batch;
  return Sched{k, stag};
}
// schedules measured per shape (kmx_ks_mul), keyed by the call's shape
struct SchedKey {
  int variant, batch, lf, lg, b, iw;
  unsigned flags;
  int dev;
  bool operator<(const SchedKey& o) const {
    const int x[7] = {variant, batch, lf, lg, b, iw, dev}, y[7] = {o.variant, o.batch, o.lf, o.lg, o.b, o.iw, o.dev};
    for (int i = 0; i < 7; i++)
      if (x[i] != y[i]) return x[i] < y[i];
    return flags < o.flags;
  }
};
std::mutex g_sched_mu;
std::map<SchedKey, Sched> g_sched;
bool tuned_sched(const SchedKey& k, Sched* s) {
  std::lock_guard<std::mutex> lk(g_sched_mu);
  auto it = g_sched.find(k);
  if (it == g_sched.end()) return false;
  *s = it->second;
  return true;
}
// the schedule a call with this shape runs (or ran) with
Sched current_sched(const SchedKey& k) {
  if (g_prof.on || (k.flags & KMX_NO_SPLIT) || split_force() >= 0) return g_prof.on ? Sched{1, 0} : default_sched(k.batch, k.flags);
  Sched s;
  if (tuned_sched(k, &s)) return s;
  return default_sched(k.batch, k.flags);
}
int max_ways(int batch, unsigned flags) {
  if ((flags & KMX_NO_SPLIT) || split_force() == 0 || batch < 2) return 1;
  int m = default_sched(batch, flags).ways;
  if (split_force() < 0 && batch >= 64) m = batch < SPLIT_MAX ? batch : SPLIT_MAX;
  return m;
}

// part i of a K-way split: pairs [start, start + size)
void split_part(int batch, int k, int i, int* start, int* size) {
  const int q = batch / k, r = batch % k;
  *start = i * q + (i < r ? i : r);
  *size = q + (i < r ? 1 : 0);
}

struct SplitCtx {
  cudaStream_t st[SPLIT_MAX] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[SPLIT_MAX] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t packed[SPLIT_MAX] = {nullptr, nullptr, nullptr, nullptr};
  int dev = -1;
};
thread_local SplitCtx g_split;

SplitCtx& split_ctx(int* rc) {
  *rc = KMX_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { *rc = KMX_ECUDA; return g_split; }
  if (g_split.fork && g_split.dev == dev) return g_split;
  if (cudaEventCreateWithFlags(&g_split.fork, cudaEventDisableTiming) != cudaSuccess) *rc = KMX_ECUDA;
  for (int i = 1; i < SPLIT_MAX && !*rc; i++)
    if (cudaStreamCreateWithFlags(&g_split.st[i], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g_split.join[i], cudaEventDisableTiming) != cudaSuccess)
      *rc = KMX_ECUDA;
  for (int i = 0; i < SPLIT_MAX && !*rc; i++)
    if (cudaEventCreateWithFlags(&g_split.packed[i], cudaEventDisableTiming) != cudaSuccess) *rc = KMX_ECUDA;
  g_split.dev = dev;
  return g_split;
}

// workspace of a K-way split: a 256-byte header (the shared error flag) and
// the K parts' workspaces
size_t split_ws_layout(int variant, int batch, int lf, int lg, int b, int iw, unsigned flags, int k,
                       size_t off[SPLIT_MAX], KsPlan* parts) {
  size_t o = 256;
  for (int i = 0; i < k; i++) {
    int s0, n;
    split_part(batch, k, i, &s0, &n);
    if (make_plan(parts[i], variant, n, lf, lg, b, iw, flags)) return 0;
    off[i] = o;
    o += align256(parts[i].total);
  }
  return o;
}

}  // namespace

extern "C" {

int kmx_ks_params(int variant, int len_f, int len_g, int coeff_bits, unsigned flags, int64_t* out8) {
  KsPlan p;
  int rc = make_plan(p, variant, 1, len_f, len_g, coeff_bits, 0, flags);
  if (rc) return rc;
  out8[0] = p.e; out8[1] = p.N1; out8[2] = p.N2; out8[3] = p.N4;
  out8[4] = p.safe; out8[5] = p.out_len; out8[6] = p.mf; out8[7] = p.mg;
  return KMX_OK;
}

int kmx_ks_out_words(int len_f, int len_g, int coeff_bits, unsigned flags) {
  KsPlan p;
  int rc = make_plan(p, 1, 1, len_f, len_g, coeff_bits, 0, flags);
  return rc ? rc : p.out_words_min;
}

size_t kmx_ks_workspace_bytes(int variant, int batch, int len_f, int len_g, int coeff_bits, unsigned flags) {
  KsPlan p;
  if (make_plan(p, variant, batch, len_f, len_g, coeff_bits, 0, flags)) return 0;
  size_t best = p.total;
  for (int k = 2; k <= max_ways(batch, flags); k++) {
    KsPlan parts[SPLIT_MAX];
    size_t off[SPLIT_MAX];
    const size_t sp = split_ws_layout(variant, batch, len_f, len_g, coeff_bits, 0, flags, k, off, parts);
    if (!sp) return 0;
    if (sp > best) best = sp;
  }
  return best;
}

static int run_sched(const Sched& sc0, const KsPlan& p, int variant, int batch, int len_f, int len_g, int coeff_bits,
                     int in_words, unsigned flags, const uint32_t* f, const uint32_t* g, uint32_t* h, int out_words,
                     void* workspace, size_t ws_bytes, cudaStream_t st);

int kmx_ks_mul(int variant, int batch, int len_f, int len_g, int coeff_bits, const uint32_t* f,
               const uint32_t* g, int in_words, uint32_t* h, int out_words, void* workspace,
               size_t ws_bytes, unsigned flags, void* stream) {
  KsPlan p;
  int rc = make_plan(p, variant, batch, len_f, len_g, coeff_bits, in_words, flags);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const SchedKey key{variant, batch, len_f, len_g, coeff_bits, p.in_words, flags, cur_dev()};
  const bool tune = !g_prof.on && !(flags & (KMX_NO_SPLIT | KMX_NO_TUNE)) && split_force() < 0 && batch >= 64;
  Sched sc0;
  if (!tune || tuned_sched(key, &sc0)) {
    if (!tune) sc0 = current_sched(key);
    return run_sched(sc0, p, variant, batch, len_f, len_g, coeff_bits, in_words, flags, f, g, h, out_words,
                     workspace, ws_bytes, st);
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return run_sched(default_sched(batch, flags), p, variant, batch, len_f, len_g, coeff_bits, in_words, flags, f, g,
                     h, out_words, workspace, ws_bytes, st);
  // first call of this shape: time every schedule (one warm-up run each, which
  // also settles the tensor-core plan of its part sizes, then one timed run)
  // and keep the fastest; every run writes the same bit-exact output
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return KMX_ECUDA;
  float best_ms = 1e30f;
  int best = 0, nl = 0, last = -1;
  for (int i = 0; i < NSCHED; i++) {
    const Sched c = SCHEDS[i];
    if (c.ways > batch || (c.ways > 1 && batch < 64)) continue;
    if ((rc = run_sched(c, p, variant, batch, len_f, len_g, coeff_bits, in_words, flags, f, g, h, out_words, workspace,
                        ws_bytes, st)))
      break;
    cudaEventRecord(e0, st);
    if ((rc = run_sched(c, p, variant, batch, len_f, len_g, coeff_bits, in_words, flags, f, g, h, out_words, workspace,
                        ws_bytes, st)))
      break;
    cudaEventRecord(e1, st);
    last = i;
    if (cudaEventSynchronize(e1) != cudaSuccess) { rc = KMX_ECUDA; break; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_ms) { best_ms = ms; best = i; nl = g_launches; }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc) return rc;
  {
    std::lock_guard<std::mutex> lk(g_sched_mu);
    g_sched[key] = SCHEDS[best];
  }
  if (getenv("KMX_TC_VERBOSE") && atoi(getenv("KMX_TC_VERBOSE")))
    fprintf(stderr, "kmx schedule: variant=%d batch=%d len=%d,%d b=%d -> %d ways%s (%.4f ms)\n", variant, batch, len_f,
            len_g, coeff_bits, SCHEDS[best].ways, SCHEDS[best].stagger ? " staggered" : "", best_ms);
  // leave the workspace as the chosen schedule lays it out (MulStats reads it)
  if (best != last &&
      (rc = run_sched(SCHEDS[best], p, variant, batch, len_f, len_g, coeff_bits, in_words, flags, f, g, h, out_words,
                      workspace, ws_bytes, st)))
    return rc;
  g_launches = nl;
  return KMX_OK;
}

static int run_sched(const Sched& sc0, const KsPlan& p, int variant, int batch, int len_f, int len_g, int coeff_bits,
                     int in_words, unsigned flags, const uint32_t* f, const uint32_t* g, uint32_t* h, int out_words,
                     void* workspace, size_t ws_bytes, cudaStream_t st) {
  int rc = KMX_OK;
  if (sc0.ways <= 1) return run_plan(p, f, g, h, out_words, workspace, ws_bytes, st);
  // K parts on K streams (fork / join by events; captured as parallel graph
  // branches): one part's latency-bound stages overlap another's tensor-core
  // multiply
  const int k = sc0.ways;
  KsPlan parts[SPLIT_MAX];
  size_t off[SPLIT_MAX];
  const size_t need = split_ws_layout(variant, batch, len_f, len_g, coeff_bits, in_words, flags, k, off, parts);
  if (!need || ws_bytes < need || !workspace) return KMX_EINVAL;
  if (out_words < p.out_words_min) return KMX_EINVAL;
  SplitCtx& sc = split_ctx(&rc);
  if (rc) return rc;
  uint32_t* hdr = (uint32_t*)workspace;  // the shared error flag (read by kmx_ws_status)
  const int stagger = sc0.stagger;  // part i starts when part i-1's pack is done
  if (cudaMemsetAsync(hdr, 0, 4, st) != cudaSuccess) return KMX_ECUDA;
  if (cudaEventRecord(sc.fork, st) != cudaSuccess) return KMX_ECUDA;
  int nl = 0;
  for (int i = 0; i < k; i++) {
    int s0, n;
    split_part(batch, k, i, &s0, &n);
    const size_t fo = (size_t)s0 * len_f * p.in_words, go = (size_t)s0 * len_g * p.in_words;
    const size_t ho = (size_t)s0 * p.out_len * out_words;
    if (i && cudaStreamWaitEvent(sc.st[i], stagger ? sc.packed[i - 1] : sc.fork, 0) != cudaSuccess) return KMX_ECUDA;
    if ((rc = run_plan(parts[i], f + fo, g + go, h + ho, out_words, (char*)workspace + off[i], parts[i].total,
                       i ? sc.st[i] : st, hdr, stagger ? sc.packed[i] : nullptr)))
      return rc;
    nl += g_launches;
  }
  g_launches = nl;
  for (int i = 1; i < k; i++) {
    if (cudaEventRecord(sc.join[i], sc.st[i]) != cudaSuccess) return KMX_ECUDA;
    if (cudaStreamWaitEvent(st, sc.join[i], 0) != cudaSuccess) return KMX_ECUDA;
  }
  return KMX_OK;
}

int kmx_ws_status(void* workspace, void* stream) {
  uint32_t fl = 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemcpyAsync(&fl, workspace, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess) return KMX_ECUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return KMX_ECUDA;
  if (fl) cudaMemsetAsync(workspace, 0, 4, st);
  return status_from_flag(fl);
}

int kmx_ws_limb_products(void* workspace, int variant, int batch, int len_f, int len_g, int coeff_bits,
                         unsigned flags, uint64_t* out, void* stream) {
  KsPlan p;
  int rc = make_plan(p, variant, batch, len_f, len_g, coeff_bits, 0, flags);
  if (rc) return rc;
  const Sched used = current_sched(SchedKey{variant, batch, len_f, len_g, coeff_bits, p.in_words, flags, cur_dev()});
  if (used.ways > 1) {  // the parts' workspaces after a 256-byte header
    const int k = used.ways;
    KsPlan parts[SPLIT_MAX];
    size_t off[SPLIT_MAX];
    if (!split_ws_layout(variant, batch, len_f, len_g, coeff_bits, 0, flags, k, off, parts)) return KMX_EINVAL;
    uint64_t tot = 0;
    for (int i = 0; i < k; i++) {
      uint64_t t = 0;
      if ((rc = kmx_ws_limb_products((char*)workspace + off[i], variant, parts[i].batch, len_f, len_g, coeff_bits,
                                     flags | KMX_NO_SPLIT, &t, stream)))
        return rc;
      tot += t;
    }
    *out = tot;
    return KMX_OK;
  }
  std::vector<uint32_t> meta((size_t)batch * p.P * 4);
  cudaStream_t st = (cudaStream_t)stream;
  if (!meta.empty()) {
    if (cudaMemcpyAsync(meta.data(), (char*)workspace + p.off_meta, meta.size() * 4, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return KMX_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return KMX_ECUDA;
  }
  uint64_t tot = 0;
  for (int pr = 0; pr < batch; pr++)
    for (int s = 0; s < p.P; s++) {
      const uint64_t bf = meta[(size_t)pr * 4 * p.P + 2 * s + 1];
      const uint64_t bg = meta[(size_t)pr * 4 * p.P + 2 * (p.P + s) + 1];
      tot += ((bf + 63) / 64) * ((bg + 63) / 64);
    }
  *out = tot;
  return KMX_OK;
}

int kmx_ks_mul_host(int variant, int batch, int len_f, int len_g, int coeff_bits, const uint32_t* f,
                    const uint32_t* g, int in_words, uint32_t* h, int out_words, unsigned flags,
                    uint64_t* limb_products64) {
  KsPlan p;
  int rc = make_plan(p, variant, batch, len_f, len_g, coeff_bits, in_words, flags);
  if (rc) return rc;
  if (out_words < p.out_words_min) return KMX_EINVAL;
  HostCtx* c = host_ctx(&rc);
  if (!c) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  const size_t fb = (size_t)batch * len_f * p.in_words * 4, gb = (size_t)batch * len_g * p.in_words * 4;
  const size_t hb = (size_t)batch * p.out_len * out_words * 4;
  if (!limb_products64 && batch >= 2) {
    // chunks of >= ~chunk_mb MB of output (KMX_HOST_CHUNK_MB, default 4), at most HOST_MAX_CHUNKS
    static const int chunk_mb = getenv("KMX_HOST_CHUNK_MB") ? atoi(getenv("KMX_HOST_CHUNK_MB")) : 4;
    size_t nch = hb / ((size_t)(chunk_mb > 0 ? chunk_mb : 2) << 20);
    if (nch > (size_t)HOST_MAX_CHUNKS) nch = HOST_MAX_CHUNKS;
    if (nch > (size_t)batch) nch = batch;
    static const int pipe = getenv("KMX_HOST_PIPE") ? atoi(getenv("KMX_HOST_PIPE")) : 1;
    if (nch >= 2)
      return pipe ? ks_mul_host_streams(p, c, f, g, h, out_words, (int)nch)
                  : ks_mul_host_pipelined(p, c, f, g, h, out_words, (int)nch);
  }
  if (!c->st && cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
  if ((rc = ensure(*c, 0, fb + gb + 256))) return rc;
  if ((rc = ensure(*c, 1, hb))) return rc;
  if ((rc = ensure(*c, 2, p.total))) return rc;
  uint32_t* df = (uint32_t*)c->buf[0];
  uint32_t* dg = (uint32_t*)((char*)c->buf[0] + align256(fb));
  if (batch == 0) return KMX_OK;
  if (cudaMemcpyAsync(df, f, fb, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return KMX_ECUDA;
  if (cudaMemcpyAsync(dg, g, gb, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return KMX_ECUDA;
  rc = run_plan(p, df, dg, (uint32_t*)c->buf[1], out_words, c->buf[2], c->cap[2], c->st);
  if (rc) return rc;
  if (cudaMemcpyAsync(h, c->buf[1], hb, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return KMX_ECUDA;
  rc = kmx_ws_status(c->buf[2], c->st);
  if (rc == KMX_OK && limb_products64)
    rc = kmx_ws_limb_products(c->buf[2], variant, batch, len_f, len_g, coeff_bits, flags | KMX_NO_SPLIT,
                              limb_products64, c->st);
  return rc;
}


// ---------------------------------------------------------- (Z/nZ)[x] front end
// kronmul.modpoly.mod_mul (modpoly.py:95-115): lift with b = bitlen(n-1)
// (:103-104), run the KS variant, reduce every coefficient mod n (:115).
static int mod_plan(KsPlan& p, int variant, int batch, int lf, int lg, uint64_t n) {
  if (n < 2) return KMX_EINVAL;  // modpoly.py:50-51
  int b = bitlen_u64(n - 1);
  if (b < 1) b = 1;              // max(1, (n-1).bit_length()) (:104)
  int rc = make_plan(p, variant, batch, lf, lg, b, 2, 0);
  if (rc) return rc;
  return p.out_words_min <= 8 ? KMX_OK : KMX_EINVAL;
}
static size_t mod_prod_bytes(const KsPlan& p) { return (size_t)p.batch * p.out_len * p.out_words_min * 4; }

size_t kmx_mod_workspace_bytes(int variant, int batch, int len_f, int len_g, uint64_t modulus) {
  KsPlan p;
  if (mod_plan(p, variant, batch, len_f, len_g, modulus)) return 0;
  return align256(p.total) + align256(mod_prod_bytes(p));
}

int kmx_mod_mul(int variant, int batch, int len_f, int len_g, uint64_t modulus, const uint64_t* f,
                const uint64_t* g, uint64_t* h, void* workspace, size_t ws_bytes, void* stream) {
  KsPlan p;
  int rc = mod_plan(p, variant, batch, len_f, len_g, modulus);
  if (rc) return rc;
  if (ws_bytes < align256(p.total) + align256(mod_prod_bytes(p)) || !workspace) return KMX_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* prod = (uint32_t*)((char*)workspace + align256(p.total));
  rc = run_plan(p, (const uint32_t*)f, (const uint32_t*)g, prod, p.out_words_min, workspace, p.total, st);
  if (rc || batch == 0) return rc;
  ModRedArgs a;
  memset(&a, 0, sizeof a);
  a.prod = prod; a.ow = p.out_words_min; a.count = (long long)batch * p.out_len;
  a.n = modulus;
  unsigned __int128 t = 1 % modulus;
  for (int q = 0; q < 8; q++) { a.tpow[q] = (unsigned long long)t; t = (t << 32) % modulus; }
  a.out = (unsigned long long*)h;
  a.f = (const unsigned long long*)f; a.nf = (long long)batch * len_f;
  a.g = (const unsigned long long*)g; a.ng = (long long)batch * len_g;
  a.err = (uint32_t*)((char*)workspace + p.off_err);
  prof_begin(5, st);
  if (launch_modred(a, st) != cudaSuccess) return KMX_ECUDA;
  prof_end(5, st);
  g_launches++;
  return KMX_OK;
}

int kmx_mod_mul_host(int variant, int batch, int len_f, int len_g, uint64_t modulus, const uint64_t* f,
                     const uint64_t* g, uint64_t* h, uint64_t* limb_products64) {
  KsPlan p;
  int rc = mod_plan(p, variant, batch, len_f, len_g, modulus);
  if (rc) return rc;
  HostCtx* c = host_ctx(&rc);
  if (!c) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  if (batch == 0) return KMX_OK;
  const size_t fb = (size_t)batch * len_f * 8, gb = (size_t)batch * len_g * 8;
  const size_t hb = (size_t)batch * p.out_len * 8;
  const size_t wb = align256(p.total) + align256(mod_prod_bytes(p));
  if (!c->st && cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
  if ((rc = ensure(*c, 0, align256(fb) + gb + 256))) return rc;
  if ((rc = ensure(*c, 1, hb))) return rc;
  if ((rc = ensure(*c, 2, wb))) return rc;
  uint64_t* df = (uint64_t*)c->buf[0];
  uint64_t* dg = (uint64_t*)((char*)c->buf[0] + align256(fb));
  if (cudaMemcpyAsync(df, f, fb, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return KMX_ECUDA;
  if (cudaMemcpyAsync(dg, g, gb, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return KMX_ECUDA;
  rc = kmx_mod_mul(variant, batch, len_f, len_g, modulus, df, dg, (uint64_t*)c->buf[1], c->buf[2], c->cap[2], c->st);
  if (rc) return rc;
  if (cudaMemcpyAsync(h, c->buf[1], hb, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return KMX_ECUDA;
  rc = kmx_ws_status(c->buf[2], c->st);
  if (rc == KMX_OK && limb_products64)  // the KS workspace leads the mod workspace
    rc = kmx_ws_limb_products(c->buf[2], variant, batch, len_f, len_g, p.b, KMX_NO_SPLIT, limb_products64, c->st);
  return rc;
}

// ------------------------------------------------------------------ K1 alone
// kronmul.pack.pack / pack_reversed / pack_negated / pack_negated_reversed
// (pack.py:79-110) for a batch of coefficient vectors at one width: K1 by
// itself, writing |value| as out_limbs little-endian limbs and [sign, bitlen]
// per vector.
int kmx_pack_limbs(int len, int width_bits, int coeff_bits) {
  if (len < 1 || width_bits < 1 || coeff_bits < 1) return KMX_EINVAL;
  const long long bits = (long long)width_bits * (len - 1) + coeff_bits + 2;
  if ((bits + 31) / 32 > (1LL << 28)) return KMX_EINVAL;
  return (int)((bits + 31) / 32);
}

int kmx_pack(int kind, int batch, int len, int width_bits, int coeff_bits, const uint32_t* coeffs, int in_words,
             uint32_t* out, int out_limbs, uint32_t* meta, void* workspace, size_t ws_bytes, void* stream) {
  if (kind < 0 || kind > 3 || batch < 0 || in_words < (coeff_bits + 31) / 32) return KMX_EINVAL;
  const int m = kmx_pack_limbs(len, width_bits, coeff_bits);
  if (m < 0) return m;
  if (2LL * width_bits < coeff_bits) return KMX_EINVAL;  // pack.py:55-59
  if (out_limbs < m || (out_limbs & 3) || ws_bytes < 256 || !workspace) return KMX_EINVAL;
  if (((uintptr_t)out & 15) || !meta) return KMX_EINVAL;  // K1 writes 16-byte limb quads
  g_launches = 0;
  if (batch == 0) return KMX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* err = (uint32_t*)workspace;
  if (cudaMemsetAsync(err, 0, 4, st) != cudaSuccess) return KMX_ECUDA;
  // limbs past m are not written by K1: clear the caller's padding
  if (out_limbs > m &&
      cudaMemset2DAsync(out + m, (size_t)out_limbs * 4, 0, (size_t)(out_limbs - m) * 4, batch, st) != cudaSuccess)
    return KMX_ECUDA;
  PackArgs pa;
  memset(&pa, 0, sizeof pa);
  pa.nops = 1; pa.N = width_bits; pa.b = coeff_bits; pa.in_words = in_words; pa.err = err;
  PackOp& o = pa.op[0];
  o.coeffs = coeffs; o.coeff_pair_stride = (long long)len * in_words; o.len = len; o.kind = kind;
  o.out = out; o.out_pair_stride = out_limbs; o.meta = meta; o.meta_pair_stride = 2; o.m = m; o.validate = 1;
  if (launch_pack(pa, batch, st) != cudaSuccess) return KMX_ECUDA;
  g_launches = 1;
  return KMX_OK;
}

int kmx_pack_host(int kind, int batch, int len, int width_bits, int coeff_bits, const uint32_t* coeffs, int in_words,
                  uint32_t* out, int out_limbs, uint32_t* meta) {
  const int m = kmx_pack_limbs(len, width_bits, coeff_bits);
  if (m < 0) return m;
  if (out_limbs & 3) return KMX_EINVAL;
  if (batch <= 0) return batch < 0 ? KMX_EINVAL : KMX_OK;
  int rc;
  HostCtx* c = host_ctx(&rc);
  if (!c) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->st && cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
  const size_t cb = (size_t)batch * len * in_words * 4, ob = (size_t)batch * out_limbs * 4, mb = (size_t)batch * 8;
  if ((rc = ensure(*c, 0, cb))) return rc;
  if ((rc = ensure(*c, 1, align256(ob) + mb))) return rc;
  if ((rc = ensure(*c, 2, 256))) return rc;
  uint32_t* dm = (uint32_t*)((char*)c->buf[1] + align256(ob));
  if (cudaMemcpyAsync(c->buf[0], coeffs, cb, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return KMX_ECUDA;
  rc = kmx_pack(kind, batch, len, width_bits, coeff_bits, (const uint32_t*)c->buf[0], in_words, (uint32_t*)c->buf[1],
                out_limbs, dm, c->buf[2], c->cap[2], c->st);
  if (rc) return rc;
  if (cudaMemcpyAsync(out, c->buf[1], ob, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return KMX_ECUDA;
  if (meta && cudaMemcpyAsync(meta, dm, mb, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return KMX_ECUDA;
  return kmx_ws_status(c->buf[2], c->st);
}

size_t kmx_reconstruct_workspace_bytes(int batch, int count, int dwords) {
  if (batch < 0 || count < 1 || dwords < 1) return 0;
  size_t o = 256 + align256((size_t)batch * 2 * (count + 1) * dwords * 4);
  if (dwords > 17) o += align256(wide_recon_scratch_words(batch, 1, dwords) * 4);  // kmx_wide.cu
  return o;
}

int kmx_reconstruct(int batch, int count, int width_bits, const uint32_t* fwd, const uint32_t* rev, int dwords,
                    uint32_t* h, int hwords, void* workspace, size_t ws_bytes, uint8_t* carries, void* stream) {
  // The reconstruction kernel reads both streams from one digit buffer; the
  // standalone entry takes them as two arrays, so stage them in the
  // workspace: [batch][2][count+1][dwords] plus the error word.
  if (batch < 0 || count < 1 || width_bits < 1 || dwords < (width_bits + 31) / 32 ||
      hwords < (2 * width_bits + 31) / 32)
    return KMX_EINVAL;
  const size_t slot = (size_t)(count + 1) * dwords;
  const size_t need = kmx_reconstruct_workspace_bytes(batch, count, dwords);
  if (ws_bytes < need) return KMX_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* err = (uint32_t*)workspace;
  uint32_t* db = (uint32_t*)((char*)workspace + 256);
  g_launches = 0;
  if (cudaMemsetAsync(err, 0, 4, st) != cudaSuccess) return KMX_ECUDA;
  if (cudaMemcpy2DAsync(db, 2 * slot * 4, fwd, slot * 4, slot * 4, batch, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return KMX_ECUDA;
  if (cudaMemcpy2DAsync(db + slot, 2 * slot * 4, rev, slot * 4, slot * 4, batch, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return KMX_ECUDA;
  ReconArgs ra;
  memset(&ra, 0, sizeof ra);
  ra.s[0] = ReconStream{0, 1, count, 0, 1};
  ra.ns = 1; ra.batch = batch; ra.W = width_bits;
  ra.dbuf = db; ra.dwords = dwords; ra.dslot_stride = (long long)slot; ra.dslots_pair = 2;
  ra.h = h; ra.out_words = hwords; ra.h_pair_stride = (long long)count * hwords; ra.err = err;
  ra.carries = carries;
  cudaError_t e = dwords > 17 ? launch_wide_recon(ra, (uint32_t*)((char*)workspace + 256 +
                                                                 align256((size_t)batch * 2 * slot * 4)), st)
                              : launch_recon(ra, st);
  g_launches = 1;
  return cuda_rc(e);
}

int kmx_reconstruct_host(int batch, int count, int width_bits, const uint32_t* fwd, const uint32_t* rev,
                         int dwords, uint32_t* h, int hwords, uint8_t* carries) {
  if (batch < 0 || count < 1 || dwords < 1 || hwords < 1) return KMX_EINVAL;
  if (batch == 0) return KMX_OK;
  int rc;
  HostCtx* c = host_ctx(&rc);
  if (!c) return rc;
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->st && cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) return KMX_ECUDA;
  const size_t db = (size_t)batch * (count + 1) * dwords * 4;
  const size_t hb = (size_t)batch * count * hwords * 4;
  const size_t cb = (size_t)batch * (2 * count + 1);
  const size_t wsb = kmx_reconstruct_workspace_bytes(batch, count, dwords);
  if ((rc = ensure(*c, 0, 2 * align256(db) + align256(cb)))) return rc;
  if ((rc = ensure(*c, 1, hb))) return rc;
  if ((rc = ensure(*c, 2, wsb))) return rc;
  uint32_t* dfw = (uint32_t*)c->buf[0];
  uint32_t* drv = (uint32_t*)((char*)c->buf[0] + align256(db));
  uint8_t* dca = (uint8_t*)((char*)c->buf[0] + 2 * align256(db));
  if (cudaMemcpyAsync(dfw, fwd, db, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return KMX_ECUDA;
  if (cudaMemcpyAsync(drv, rev, db, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return KMX_ECUDA;
  rc = kmx_reconstruct(batch, count, width_bits, dfw, drv, dwords, (uint32_t*)c->buf[1], hwords, c->buf[2],
                       c->cap[2], carries ? dca : nullptr, c->st);
  if (rc) return rc;
  if (cudaMemcpyAsync(h, c->buf[1], hb, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return KMX_ECUDA;
  if (carries && cudaMemcpyAsync(carries, dca, cb, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return KMX_ECUDA;
  return kmx_ws_status(c->buf[2], c->st);
}

double kmx_imad_peak(int iters) { return measure_imad_peak(iters > 0 ? iters : 4096); }

double kmx_tc_peak(int iters) { return measure_tc_peak(iters > 0 ? iters : 2000); }

double kmx_tc_peak_n(int n, int iters) { return measure_tc_peak_shape(n, iters > 0 ? iters : 2000); }

int kmx_mul_plan(int variant, int batch, int len_f, int len_g, int coeff_bits, unsigned flags, int64_t* out8) {
  KsPlan p;
  int rc = make_plan(p, variant, batch, len_f, len_g, coeff_bits, 0, flags);
  if (rc) return rc;
  long long o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long nprod = (long long)batch * p.P;
  if (p.kara) o[0] = 3, o[1] = kara_levels(p.mf, p.mg);  // Karatsuba over the engines
  else if (use_tensor_mul(p.mf, p.mg) && !use_tcj(p.mf, p.mg, nprod)) tc_plan_info(p.mf, p.mg, nprod, o);
  else if (use_tensor_mul(p.mf, p.mg)) o[0] = 2;  // chunked single-tile kernel
  for (int i = 0; i < 8; i++) out8[i] = o[i];
  return KMX_OK;
}

int kmx_mul_engine(int variant, int len_f, int len_g, int coeff_bits, unsigned flags) {
  KsPlan p;
  int rc = make_plan(p, variant, 1, len_f, len_g, coeff_bits, 0, flags);
  if (rc) return rc;
  // Karatsuba levels: the engine of the leaves (the split halves)
  int ma = p.mf, mb = p.mg;
  while (!mul_engine_takes(ma, mb)) {
    const int mx = ma > mb ? ma : mb, h = (((mx + 1) / 2) + 3) & ~3;  // kmx_kara.cu node()
    if ((ma < mb ? ma : mb) > h) ma = mb = h + 1;
    else if (ma >= mb) ma = h;
    else mb = h;
  }
  return use_tensor_mul(ma, mb) ? 1 : 0;
}

int kmx_mul_karatsuba_levels(int variant, int batch, int len_f, int len_g, int coeff_bits, unsigned flags) {
  KsPlan p;
  int rc = make_plan(p, variant, batch, len_f, len_g, coeff_bits, 0, flags);
  if (rc) return rc;
  return p.kara ? kara_levels(p.mf, p.mg) : 0;
}

const char* kmx_error_string(int code) {
  switch (code) {
    case KMX_OK: return "ok";
    case KMX_EINVAL: return "invalid argument (ValueError)";
    case KMX_ERECON: return "overlapped digit streams are inconsistent (ReconstructionError)";
    case KMX_EINEXACT: return "inexact halving/shift or value does not fit its digits (ValueError)";
    case KMX_ECUDA: return "CUDA error";
    case KMX_ENOMEM: return "device out of memory";
    default: return "unknown error";
  }
}

int kmx_last_launch_count(void) { return g_launches; }

void kmx_prof_enable(int on) { g_prof.on = on != 0; }

int kmx_prof_read(float* ms, int nslots) {
  int n = 0;
  for (int i = 0; i < nslots && i < 6; i++) {
    ms[i] = 0.f;
    if (!g_prof.on || !g_prof.created || !g_prof.used[i]) continue;
    if (cudaEventSynchronize(g_prof.ev[i][1]) != cudaSuccess) return KMX_ECUDA;
    if (cudaEventElapsedTime(&ms[i], g_prof.ev[i][0], g_prof.ev[i][1]) != cudaSuccess) return KMX_ECUDA;
    n++;
  }
  return n;
}

}  // extern "C"
