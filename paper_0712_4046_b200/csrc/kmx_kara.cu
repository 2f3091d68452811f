// kmx_kara.cu -- Karatsuba levels above the batched multiply engines (the
// reference's _karatsuba_int, bignat.py:344-363, dispatched by _mul_int
// :366-371), batched over all products of a launch.
//
// One level, operands a = a0 + a1 X, b = b0 + b1 X, X = 2^(32h),
// h = ceil(max(ma, mb) / 2):
//   balanced (min(ma, mb) > h): three products
//     z0 = a0 b0, z2 = a1 b1, z1 = (a0 + a1)(b0 + b1)
//     a b = z0 + (z1 - z0 - z2) X + z2 X^2
//   unbalanced (the shorter operand fits in h limbs): two products
//     z0 = a0 b, z1 = a1 b,  a b = z0 + z1 X.
// The sub-products are strided views of the operands (no copies) except the
// half sums, and recurse until the multiply engine takes them: the tcgen05
// byte convolution stages whole operands in shared memory, so this is what
// keeps long operands (c4 ks1, config-5 n = 8192 ks1) on the tensor cores,
// and above a measured size it is also faster there (fewer MACs).
//
// The sums and the recombination are one kernel pair, a "linear combination
// normalizer": out = sum_t sign_t * term_t * 2^(32 off_t), where each term is
// a product in the engines' output format (normalized 32-bit limbs plus band
// spills folded in at band starts, kmx_finish.cuh).  Every output limb is a
// small signed 64-bit sum; each thread resolves its 8 limbs with carry-in 0,
// which leaves digits R (256 bits) and a carry c0, and the carry out for a
// carry-in c is c0 + [R + c >= 2^256] - [R + c < 0].  That map is stored as
// (R, 2^256 - R, out(-), out(0), out(+)) with the thresholds saturated at
// 2^62; maps compose associatively (g o f keeps f's thresholds and maps its
// three outputs through g), so a block scan plus a chunk-level pass resolve
// every carry chain exactly:
//   k_lc_map    one map per 2048-limb chunk (block reduction);
//   k_lc_apply  chunk carry-in from the preceding chunk maps, block scan,
//               final digits, zero check above the output length.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

namespace {

constexpr int LC_T = 256;             // threads per chunk
constexpr int LC_V = 8;               // limbs per thread
constexpr int LC_CH = LC_T * LC_V;    // limbs per chunk
constexpr long long LC_SAT = 1LL << 62;

struct LcMap {
  long long R, D, om, o0, op;
};

__device__ __forceinline__ long long lc_apply(const LcMap& f, long long c) {
  return c < -f.R ? f.om : (c >= f.D ? f.op : f.o0);
}
// g after f
__device__ __forceinline__ LcMap lc_compose(const LcMap& f, const LcMap& g) {
  return LcMap{f.R, f.D, lc_apply(g, f.om), lc_apply(g, f.o0), lc_apply(g, f.op)};
}
__device__ __forceinline__ LcMap lc_shfl_up(const LcMap& m, int d) {
  return LcMap{__shfl_up_sync(0xffffffffu, m.R, d), __shfl_up_sync(0xffffffffu, m.D, d),
               __shfl_up_sync(0xffffffffu, m.om, d), __shfl_up_sync(0xffffffffu, m.o0, d),
               __shfl_up_sync(0xffffffffu, m.op, d)};
}

// the signed sum at output limb i of product z
__device__ __forceinline__ long long lc_limb(const LcArgs& a, long long z, long long i) {
  long long s = 0;
#pragma unroll
  for (int t = 0; t < LC_MAXT; t++) {
    if (t >= a.nt) break;
    const LcTerm& T = a.t[t];
    const long long j = i - T.off;
    if (j < 0 || j >= T.len) continue;
    long long v = (long long)__ldg(T.p + z * T.stride + j);
    if (T.spill) {  // band spills fold in at band starts (kmx_finish.cuh)
      const long long* sp =
          reinterpret_cast<const long long*>(T.spill) + z * (T.spill_stride ? T.spill_stride : T.nbands * 2LL);
      if (j > 0 && (j & 255) == 0 && (j >> 8) <= T.nbands) v += sp[((j >> 8) - 1) * 2];
      if (j > 1 && (j & 255) == 1 && (j >> 8) <= T.nbands) v += sp[((j >> 8) - 1) * 2 + 1];
    }
    int sg = T.sign;
    if (T.smeta) {
      const uint32_t* m = T.smeta + z * T.smeta_stride;
      if (m[0] ^ m[T.smeta_off]) sg = -sg;
    }
    s += sg > 0 ? v : -v;
  }
  return s;
}

// this thread's digits with carry-in 0 and its carry map
__device__ __forceinline__ LcMap lc_thread(const LcArgs& a, long long z, long long i0, u32 d[LC_V]) {
  long long c = 0;
#pragma unroll
  for (int v = 0; v < LC_V; v++) {
    const long long x = lc_limb(a, z, i0 + v) + c;
    d[v] = (u32)x;
    c = x >> 32;  // floor
  }
  bool hi0 = true, hiF = true;
#pragma unroll
  for (int v = 2; v < LC_V; v++) {
    hi0 &= d[v] == 0u;
    hiF &= d[v] == 0xffffffffu;
  }
  const unsigned long long x = ((unsigned long long)d[1] << 32) | d[0];
  LcMap m;
  m.R = (hi0 && x < (unsigned long long)LC_SAT) ? (long long)x : LC_SAT;
  const unsigned long long dd = 0ull - x;  // 2^64 - x (x != 0)
  m.D = (hiF && x != 0ull && dd < (unsigned long long)LC_SAT) ? (long long)dd : LC_SAT;
  m.om = c - 1;
  m.o0 = c;
  m.op = c + 1;
  return m;
}

__global__ void __launch_bounds__(LC_T) k_lc_map(LcArgs a) {
  __shared__ LcMap wm[LC_T / 32];
  const long long z = blockIdx.x / a.nchunks;
  const int ch = blockIdx.x - (int)(z * a.nchunks);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 d[LC_V];
  LcMap m = lc_thread(a, z, (long long)ch * LC_CH + (long long)threadIdx.x * LC_V, d);
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const LcMap o = lc_shfl_up(m, off);
    if (lane >= off) m = lc_compose(o, m);
  }
  if (lane == 31) wm[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    LcMap t = wm[0];
    for (int w = 1; w < LC_T / 32; w++) t = lc_compose(t, wm[w]);
    reinterpret_cast<LcMap*>(a.maps)[z * a.nchunks + ch] = t;
  }
}

__global__ void __launch_bounds__(LC_T) k_lc_apply(LcArgs a) {
  __shared__ LcMap wm[LC_T / 32];
  __shared__ long long cin_chunk;
  const long long z = blockIdx.x / a.nchunks;
  const int ch = blockIdx.x - (int)(z * a.nchunks);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    const LcMap* mp = reinterpret_cast<const LcMap*>(a.maps) + z * a.nchunks;
    long long c = 0;
    for (int k = 0; k < ch; k++) c = lc_apply(mp[k], c);
    cin_chunk = c;
  }
  const long long i0 = (long long)ch * LC_CH + (long long)threadIdx.x * LC_V;
  u32 d[LC_V];
  const LcMap m = lc_thread(a, z, i0, d);
  LcMap inc = m;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const LcMap o = lc_shfl_up(inc, off);
    if (lane >= off) inc = lc_compose(o, inc);
  }
  const LcMap exc = lc_shfl_up(inc, 1);
  if (lane == 31) wm[warp] = inc;
  __syncthreads();
  long long c = cin_chunk;
  for (int w = 0; w < warp; w++) c = lc_apply(wm[w], c);
  if (lane) c = lc_apply(exc, c);
  const long long cout = lc_apply(m, c);
  // digits = R + c (|c| small): ripple through this thread's limbs
  long long x = c;
  bool bad = false;
  u32* out = a.out + z * a.out_stride;
#pragma unroll
  for (int v = 0; v < LC_V; v++) {
    x += (long long)d[v];
    const u32 dv = (u32)x;
    x >>= 32;
    const long long i = i0 + v;
    if (i < a.out_len) out[i] = dv;
    else bad |= dv != 0u;
  }
  // the value fits in out_len limbs: nothing above it, no carry out of the top
  if (i0 + LC_V >= (long long)a.nchunks * LC_CH) bad |= cout != 0;
  if (bad && a.err) raise_err(a.err, ERR_INEXACT);
}

}  // namespace

int lc_chunks(int out_len) { return (out_len + LC_CH - 1) / LC_CH; }
size_t lc_map_bytes(long long nprod, int out_len) { return (size_t)nprod * lc_chunks(out_len) * sizeof(LcMap); }

cudaError_t launch_lincomb(const LcArgs& a0, long long nprod, cudaStream_t st) {
  LcArgs a = a0;
  a.nchunks = lc_chunks(a.out_len);
  if (nprod == 0) return cudaSuccess;
  const long long grid = nprod * a.nchunks;
  k_lc_map<<<(unsigned)grid, LC_T, 0, st>>>(a);
  k_lc_apply<<<(unsigned)grid, LC_T, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ planning
namespace {

int env_int_k(const char* n, int dflt) {
  const char* v = getenv(n);
  return v && *v ? atoi(v) : dflt;
}
size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Node {
  int ma, mb, h;
  bool leaf, balanced;
};

// Karatsuba above this many limbs (the longer operand) even where the
// multiply engine takes the whole product: KMX_KARA_MIN, default measured.
int kara_min_limbs() {
  static const int v = env_int_k("KMX_KARA_MIN", 1 << 30);
  return v;
}

Node node(int ma, int mb, int depth) {
  Node n;
  n.ma = ma;
  n.mb = mb;
  const int mx = std::max(ma, mb), mn = std::min(ma, mb);
  n.h = (((mx + 1) / 2) + 3) & ~3;  // a multiple of 4 limbs: the a1 / b1 views stay 16-byte aligned (bulk staging)
  n.balanced = mn > n.h;
  const bool engine_ok = mul_engine_takes(ma, mb);
  n.leaf = depth >= KARA_MAX_DEPTH || mn < 64 || (engine_ok && mx < kara_min_limbs());
  return n;
}

int nb_of(int ma, int mb) { return (ma + mb + 255) / 256; }
long long pstride_of(int ma, int mb) { return (long long)nb_of(ma, mb) * 256; }
int pad4(int x) { return (x + 3) & ~3; }

// child shapes of a non-leaf node
int children(const Node& n, int cm[3][2]) {
  const int h = n.h;
  if (n.balanced) {
    cm[0][0] = h; cm[0][1] = h;                        // z0
    cm[1][0] = n.ma - h; cm[1][1] = n.mb - h;          // z2
    cm[2][0] = h + 1; cm[2][1] = h + 1;                // z1 (sums)
    return 3;
  }
  if (n.ma >= n.mb) {
    cm[0][0] = h; cm[0][1] = n.mb;
    cm[1][0] = n.ma - h; cm[1][1] = n.mb;
  } else {
    cm[0][0] = n.ma; cm[0][1] = h;
    cm[1][0] = n.ma; cm[1][1] = n.mb - h;
  }
  return 2;
}

size_t node_ws(int ma, int mb, long long nprod, int depth) {
  const Node n = node(ma, mb, depth);
  if (n.leaf) return 256;  // the leaf's work counter
  int cm[3][2];
  const int nc = children(n, cm);
  size_t o = 256;
  if (n.balanced) o += 2 * al256((size_t)nprod * pad4(n.h + 1) * 4);
  size_t maps = 0;
  for (int c = 0; c < nc; c++) {
    o += al256((size_t)nprod * pstride_of(cm[c][0], cm[c][1]) * 4);
    o += al256((size_t)nprod * nb_of(cm[c][0], cm[c][1]) * 16);
  }
  maps = std::max(lc_map_bytes(nprod, n.h + 1), lc_map_bytes(nprod, ma + mb));
  o += al256(maps);
  size_t child = 0;
  for (int c = 0; c < nc; c++) child = std::max(child, node_ws(cm[c][0], cm[c][1], nprod, depth + 1));
  return o + child;
}

int node_levels(int ma, int mb, int depth) {
  const Node n = node(ma, mb, depth);
  if (n.leaf) return 0;
  int cm[3][2];
  const int nc = children(n, cm);
  int lv = 0;
  for (int c = 0; c < nc; c++) lv = std::max(lv, node_levels(cm[c][0], cm[c][1], depth + 1));
  return lv + 1;
}

cudaError_t leaf_mul(const MulArgs& base, int ma, int mb, const u32* A, long long as, const u32* B, long long bs,
                     u32* P, unsigned long long* spill, int* counter, cudaStream_t st, int* nl) {
  MulArgs m = base;
  m.A = A; m.a_stride = as; m.ma = ma;
  m.B = B; m.b_stride = bs; m.mb = mb;
  int split, cw, nbands, tr;
  mul_geometry(ma, mb, &split, &cw, &nbands, &tr);
  m.P = P; m.p_stride = (long long)nbands * cw; m.spill = spill;
  m.nbands = nbands; m.G = split; m.TI = tr;
  m.counter = counter;
  cudaError_t e;
  if (mul_engine_takes(ma, mb)) e = launch_tcmul(m, st);
  else e = launch_mul(m, st);
  (*nl)++;
  return e;
}

// product of the views (A, as, ma) x (B, bs, mb) into P (p_stride ps,
// spill[z][nbands_out][2] zeroed: normalized output)
cudaError_t node_mul(const MulArgs& base, int ma, int mb, const u32* A, long long as, const u32* B, long long bs,
                     u32* P, long long ps, unsigned long long* spill, int nbands_out, char* ws, int depth,
                     cudaStream_t st, int* nl) {
  const long long nprod = base.nprod;
  const Node n = node(ma, mb, depth);
  cudaError_t e;
  if (n.leaf) {
    // the engine writes its own spill layout (nb_of(ma, mb) bands of 256
    // limbs) which is the caller's layout too (P was sized by pstride_of)
    if ((e = cudaMemsetAsync(ws, 0, 4, st)) != cudaSuccess) return e;
    (void)ps; (void)nbands_out;
    return leaf_mul(base, ma, mb, A, as, B, bs, P, spill, reinterpret_cast<int*>(ws), st, nl);
  }
  int cm[3][2];
  const int nc = children(n, cm);
  const int h = n.h;
  char* o = ws + 256;
  u32* SA = nullptr;
  u32* SB = nullptr;
  const int sw = pad4(h + 1);
  if (n.balanced) {
    SA = reinterpret_cast<u32*>(o); o += al256((size_t)nprod * sw * 4);
    SB = reinterpret_cast<u32*>(o); o += al256((size_t)nprod * sw * 4);
  }
  u32* Z[3];
  unsigned long long* ZS[3];
  for (int c = 0; c < nc; c++) {
    Z[c] = reinterpret_cast<u32*>(o); o += al256((size_t)nprod * pstride_of(cm[c][0], cm[c][1]) * 4);
    ZS[c] = reinterpret_cast<unsigned long long*>(o); o += al256((size_t)nprod * nb_of(cm[c][0], cm[c][1]) * 16);
  }
  char* maps = o;
  o += al256(std::max(lc_map_bytes(nprod, h + 1), lc_map_bytes(nprod, ma + mb)));
  char* child = o;
  LcArgs la;
  memset(&la, 0, sizeof la);
  la.maps = maps;
  la.err = base.err;
  if (n.balanced) {
    // half sums a0 + a1, b0 + b1 (h + 1 limbs)
    for (int side = 0; side < 2; side++) {
      const u32* X = side ? B : A;
      const long long xs = side ? bs : as;
      const int mx = side ? mb : ma;
      la.nt = 2;
      la.t[0] = LcTerm{X, xs, h, 0, +1, nullptr, 0, 0, nullptr, 0, 0};
      la.t[1] = LcTerm{X + h, xs, mx - h, 0, +1, nullptr, 0, 0, nullptr, 0, 0};
      la.out = side ? SB : SA;
      la.out_stride = sw;
      la.out_len = h + 1;
      if ((e = launch_lincomb(la, nprod, st)) != cudaSuccess) return e;
      *nl += 2;
    }
    const u32* CA[3] = {A, A + h, SA};
    const u32* CB[3] = {B, B + h, SB};
    const long long CAS[3] = {as, as, sw}, CBS[3] = {bs, bs, sw};
    for (int c = 0; c < 3; c++)
      if ((e = node_mul(base, cm[c][0], cm[c][1], CA[c], CAS[c], CB[c], CBS[c], Z[c], pstride_of(cm[c][0], cm[c][1]),
                        ZS[c], nb_of(cm[c][0], cm[c][1]), child, depth + 1, st, nl)) != cudaSuccess)
        return e;
    // a b = z0 + z1 X - z0 X - z2 X + z2 X^2
    const int l0 = cm[0][0] + cm[0][1], l2 = cm[1][0] + cm[1][1], l1 = cm[2][0] + cm[2][1];
    const int nb0 = nb_of(cm[0][0], cm[0][1]), nb2 = nb_of(cm[1][0], cm[1][1]), nb1 = nb_of(cm[2][0], cm[2][1]);
    const long long p0 = pstride_of(cm[0][0], cm[0][1]), p2 = pstride_of(cm[1][0], cm[1][1]),
                    p1 = pstride_of(cm[2][0], cm[2][1]);
    la.nt = 5;
    la.t[0] = LcTerm{Z[0], p0, l0, 0, +1, ZS[0], nb0, 0, nullptr, 0, 0};
    la.t[1] = LcTerm{Z[2], p1, l1, h, +1, ZS[2], nb1, 0, nullptr, 0, 0};
    la.t[2] = LcTerm{Z[0], p0, l0, h, -1, ZS[0], nb0, 0, nullptr, 0, 0};
    la.t[3] = LcTerm{Z[1], p2, l2, h, -1, ZS[1], nb2, 0, nullptr, 0, 0};
    la.t[4] = LcTerm{Z[1], p2, l2, 2LL * h, +1, ZS[1], nb2, 0, nullptr, 0, 0};
  } else {
    const bool along_a = ma >= mb;
    const u32* CA[2] = {A, along_a ? A + h : A};
    const u32* CB[2] = {B, along_a ? B : B + h};
    for (int c = 0; c < 2; c++)
      if ((e = node_mul(base, cm[c][0], cm[c][1], CA[c], as, CB[c], bs, Z[c], pstride_of(cm[c][0], cm[c][1]), ZS[c],
                        nb_of(cm[c][0], cm[c][1]), child, depth + 1, st, nl)) != cudaSuccess)
        return e;
    la.nt = 2;
    la.t[0] = LcTerm{Z[0], pstride_of(cm[0][0], cm[0][1]), cm[0][0] + cm[0][1], 0, +1, ZS[0], nb_of(cm[0][0], cm[0][1]), 0, nullptr, 0, 0};
    la.t[1] = LcTerm{Z[1], pstride_of(cm[1][0], cm[1][1]), cm[1][0] + cm[1][1], h, +1, ZS[1],
                     nb_of(cm[1][0], cm[1][1])};
  }
  la.out = P;
  la.out_stride = ps;
  la.out_len = ma + mb;
  if ((e = launch_lincomb(la, nprod, st)) != cudaSuccess) return e;
  *nl += 2;
  // the output is normalized: no band spills for the consumer to fold in
  return cudaMemsetAsync(spill, 0, (size_t)nprod * nbands_out * 16, st);
}

}  // namespace

bool kara_used(int ma, int mb) { return !node(ma, mb, 0).leaf; }
int kara_levels(int ma, int mb) { return node_levels(ma, mb, 0); }
size_t kara_ws_bytes(int ma, int mb, long long nprod) {
  return kara_used(ma, mb) ? al256(node_ws(ma, mb, nprod, 0)) : 0;
}

cudaError_t launch_kara(const MulArgs& a, void* ws, cudaStream_t st, int* nlaunch) {
  int nl = 0;
  cudaError_t e = node_mul(a, a.ma, a.mb, a.A, a.a_stride, a.B, a.b_stride, a.P, a.p_stride, a.spill, a.nbands,
                           reinterpret_cast<char*>(ws), 0, st, &nl);
  if (nlaunch) *nlaunch = nl;
  return e;
}

}  // namespace kmx
