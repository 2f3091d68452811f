// Batched schoolbook products on the integer pipe (sm_100a).
//
// One engine serves both multiply families of the path:
//   * k_mul  -- multiprecision integer products of the packed operands
//              (bignat.mul / _classical_int, bignat.py:323-380): 32x32->64
//              limb products accumulated in 96-bit column sums, one
//              IMAD.WIDE.U32 (carry-out) + half an IADD3.X per product;
//   * k_conv -- the univariate Z[x] products of the bivariate reductions
//              (UniMul, bipoly.py:23 / oracle.uni_schoolbook :58-69):
//              int32 x int32 -> int64 column sums, one IMAD.WIDE per term.
//
// Geometry.  A warp owns a band of CW consecutive product columns; its 32
// lanes form SPLIT row-groups of LPG = 32/SPLIT lanes, each lane holding 8
// consecutive columns (CW = 8*LPG), and the row-groups split the band's rows
// into SPLIT contiguous slices (partial sums are added across groups at the
// end).  Every warp walks only the rows its own columns need (exact to an
// 8-row block), so the zero-padding work is (CW + 8)/(m + CW) instead of the
// whole CTA's span.  A CTA of 8 warps stages the operand rows/columns its
// bands need in shared memory, TR rows at a time.  The inner loop is an 8x8
// register block: per 64 limb products two broadcast LDS.128 for a and two
// LDS.128 for the sliding b window, whose two 8-word halves swap roles every
// block (no register moves).
#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

// ----------------------------------------------------------- accumulators
struct AccBig {  // 96-bit unsigned column sums
  u32 c0[8], c1[8], c2[8];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < 8; r++) c0[r] = c1[r] = c2[r] = 0u;
  }
  __device__ __forceinline__ void mac(int r, u32 a, u32 b) { mac96(c0[r], c1[r], c2[r], a, b); }
  __device__ __forceinline__ void add_from_lane(int delta) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const u32 o0 = __shfl_down_sync(0xffffffffu, c0[r], delta);
      const u32 o1 = __shfl_down_sync(0xffffffffu, c1[r], delta);
      const u32 o2 = __shfl_down_sync(0xffffffffu, c2[r], delta);
      asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
          : "+r"(c0[r]), "+r"(c1[r]), "+r"(c2[r])
          : "r"(o0), "r"(o1), "r"(o2));
    }
  }
};

struct AccI64 {  // signed 64-bit column sums
  long long s[8];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < 8; r++) s[r] = 0;
  }
  __device__ __forceinline__ void mac(int r, u32 a, u32 b) { s[r] += (long long)(int)a * (int)b; }
  __device__ __forceinline__ void add_from_lane(int delta) {
#pragma unroll
    for (int r = 0; r < 8; r++) s[r] += __shfl_down_sync(0xffffffffu, s[r], delta);
  }
};

template <class ACC>
__device__ __forceinline__ void mac_block(ACC& acc, const u32 av[8], const u32 lo[8], const u32 hi[8]) {
  // column r += a[v] * b[k_r - i_v]; window index 7 + r - v
#pragma unroll
  for (int v = 0; v < 8; v++) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int idx = 7 + r - v;
      acc.mac(r, av[v], idx < 8 ? lo[idx] : hi[idx - 8]);
    }
  }
}

__device__ __forceinline__ void lds8(u32 d[8], const u32* p) {
  const uint4 x = reinterpret_cast<const uint4*>(p)[0];
  const uint4 y = reinterpret_cast<const uint4*>(p)[1];
  d[0] = x.x; d[1] = x.y; d[2] = x.z; d[3] = x.w;
  d[4] = y.x; d[5] = y.y; d[6] = y.z; d[7] = y.w;
}

// nblk consecutive 8-row blocks: a rows at ap[0..8*nblk), window of block 0
// at bp[0..16), block t's window at bp[-8t .. -8t+16).
template <class ACC>
__device__ __forceinline__ void walk(ACC& acc, const u32* ap, const u32* bp, int nblk) {
  if (nblk <= 0) return;
  u32 wl[8], wh[8], av[8];
  lds8(wl, bp);
  lds8(wh, bp + 8);
  int t = 0;
  for (; t + 2 <= nblk; t += 2) {
    lds8(av, ap + 8 * t);
    mac_block(acc, av, wl, wh);
    lds8(wh, bp - 8 * (t + 1));      // next window = (wh_new, wl)
    lds8(av, ap + 8 * (t + 1));
    mac_block(acc, av, wh, wl);
    if (t + 2 < nblk) lds8(wl, bp - 8 * (t + 2));  // next window = (wl_new, wh)
  }
  if (t < nblk) {
    lds8(av, ap + 8 * t);
    mac_block(acc, av, wl, wh);
  }
}

struct BandGeom {
  int K0, Kw, ilo, ihi, gb_lo, gb_hi;  // global 8-row blocks [gb_lo, gb_hi) of this group
};

// Main loop shared by both kernels.  Returns with acc holding this lane's
// partial column sums (before the cross-group reduction).
template <int SPLIT, class ACC>
__device__ __forceinline__ void band_engine(ACC& acc, const u32* A, int ma, const u32* B, int mb, int K0, int TR,
                                            u32* smem, int& Kw_out) {
  constexpr int LPG = 32 / SPLIT;
  constexpr int CW = 8 * LPG;
  constexpr int CC = 8 * CW;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = lane / LPG, p = lane - grp * LPG;
  const int Kw = K0 + warp * CW;
  Kw_out = Kw;
  u32* as_ = smem;
  u32* bs_ = smem + TR;
  const int ilo = max(0, K0 - (mb - 1));
  const int ihi = min(ma - 1, K0 + CC - 1);
  // this warp's rows (8-row blocks relative to ilo) and this group's slice
  const int wlo = max(0, Kw - (mb - 1)), whi = min(ma - 1, Kw + CW - 1);
  int wb_lo = (wlo - ilo) >> 3, wb_hi = (whi - ilo + 8) >> 3;
  if (whi < wlo) wb_hi = wb_lo;
  const int qb = (wb_hi - wb_lo + SPLIT - 1) / SPLIT;
  const int gb_lo = min(wb_hi, wb_lo + grp * qb), gb_hi = min(wb_hi, gb_lo + qb);
  acc.zero();
  const int TRB = TR >> 3;
  for (int i0 = ilo; i0 <= ihi; i0 += TR) {
    for (int x = tid; x < TR; x += blockDim.x) {
      const int i = i0 + x;
      as_[x] = i < ma ? A[i] : 0u;
    }
    const int bbase = K0 - i0 - TR + 1;
    for (int x = tid; x < CC + TR; x += blockDim.x) {
      const int j = bbase + x;
      bs_[x] = (j >= 0 && j < mb) ? B[j] : 0u;
    }
    __syncthreads();
    const int cb0 = (i0 - ilo) >> 3;
    const int s = max(gb_lo, cb0), e = min(gb_hi, cb0 + TRB);
    if (s < e) {
      const int xb = (Kw - K0) + 8 * p - 8 * (s - cb0) + TR - 8;
      walk(acc, as_ + 8 * (s - cb0), bs_ + xb, e - s);
    }
    __syncthreads();
  }
  // cross-group reduction: group 0 ends with the band's column sums
#pragma unroll
  for (int st = SPLIT / 2; st >= 1; st >>= 1) acc.add_from_lane(st * LPG);
}

// ======================================================= bigint products
template <int SPLIT>
__global__ void __launch_bounds__(256) k_mul(MulArgs a) {
  extern __shared__ __align__(16) u32 smem[];
  constexpr int LPG = 32 / SPLIT;
  constexpr int CW = 8 * LPG;
  constexpr int CC = 8 * CW;
  const int nbpp = a.nbands / 8;  // CTAs per product
  const int z = blockIdx.x / nbpp;
  const int K0 = (blockIdx.x - z * nbpp) * CC;
  const u32* A = a.A + (long long)z * a.a_stride;
  const u32* B = a.B + (long long)z * a.b_stride;
  AccBig acc;
  int Kw;
  band_engine<SPLIT>(acc, A, a.ma, B, a.mb, K0, a.TI, smem, Kw);

  // ---- band normalization (group-0 lanes; others compute and discard)
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPG, p = lane - grp * LPG;
  // digit y_r = c0_r + c1_{r-1} + c2_{r-2} (< 3 * 2^32)
  u32 p_c1 = __shfl_up_sync(0xffffffffu, acc.c1[7], 1, LPG);
  u32 p_c2 = __shfl_up_sync(0xffffffffu, acc.c2[7], 1, LPG);
  u32 p_c2b = __shfl_up_sync(0xffffffffu, acc.c2[6], 1, LPG);
  if (p == 0) p_c1 = p_c2 = p_c2b = 0u;
  u32 lo[8], hi[8];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const u64 y = (u64)acc.c0[r] + (r >= 1 ? acc.c1[r - 1] : p_c1) +
                  (r >= 2 ? acc.c2[r - 2] : (r == 1 ? p_c2 : p_c2b));
    lo[r] = (u32)y;
    hi[r] = (u32)(y >> 32);
  }
  u32 hprev = __shfl_up_sync(0xffffffffu, hi[7], 1, LPG);
  if (p == 0) hprev = 0u;
  i64 zz[8];
  u32 mr[8], M = CM_IDENT;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    zz[r] = (i64)lo[r] + (r ? hi[r - 1] : hprev);
    mr[r] = cm_make(zz[r]);
    M = cm_compose(M, mr[r]);
  }
  u32 tot;
  const u32 exc = cm_seg_scan(M, LPG, nullptr, &tot);
  int c = cm_apply(exc, 0);
  u32 d[8];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    d[r] = (u32)(zz[r] + c);
    c = cm_apply(mr[r], c);
  }
  const int mp = a.ma + a.mb;
  if (grp == 0 && Kw < mp) {
    uint4* dst = reinterpret_cast<uint4*>(a.P + (long long)z * a.p_stride + Kw + 8 * p);
    dst[0] = make_uint4(d[0], d[1], d[2], d[3]);
    dst[1] = make_uint4(d[4], d[5], d[6], d[7]);
    if (p == LPG - 1) {
      const int band = Kw / CW;
      const i64 s0 = (i64)c + hi[7] + acc.c1[7] + acc.c2[6];
      unsigned long long* sp = a.spill + ((long long)z * a.nbands + band) * 2;
      sp[0] = (unsigned long long)s0;
      sp[1] = (unsigned long long)acc.c2[7];
    }
  }
}

template <int SPLIT>
static cudaError_t launch_mul_t(const MulArgs& a, cudaStream_t st) {
  const int grid = a.nprod * (a.nbands / 8);
  constexpr int CW = 8 * (32 / SPLIT);
  const size_t smem = (size_t)(2 * a.TI + 8 * CW) * sizeof(u32);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_mul<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_mul<SPLIT><<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_mul(const MulArgs& a, cudaStream_t st) {
  switch (a.G) {  // G carries SPLIT
    case 1: return launch_mul_t<1>(a, st);
    case 2: return launch_mul_t<2>(a, st);
    case 4: return launch_mul_t<4>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

void mul_geometry(int ma, int mb, int* split, int* cw, int* nbands, int* tr) {
  const int m = ma < mb ? ma : mb;
  int s = m < 1024 ? 4 : (m < 4096 ? 2 : 1);
  const int CW = 8 * (32 / s);
  const int CC = 8 * CW;
  const int mp = ma + mb;
  const int nbpp = (mp + CC - 1) / CC;
  int T = (ma + 7) & ~7;
  if (T > 1024) T = 1024;
  if (T < 8) T = 8;
  *split = s;
  *cw = CW;
  *nbands = nbpp * 8;
  *tr = T;
}

// ================================================= univariate Z[x] products
template <int SPLIT>
__global__ void __launch_bounds__(256) k_conv(ConvArgs a) {
  extern __shared__ __align__(16) u32 smem[];
  constexpr int LPG = 32 / SPLIT;
  constexpr int CW = 8 * LPG;
  constexpr int CC = 8 * CW;
  const int nbpp = a.nbands / 8;
  const int z = blockIdx.x / nbpp;
  const int K0 = (blockIdx.x - z * nbpp) * CC;
  const u32* A = reinterpret_cast<const u32*>(a.A + (long long)z * a.a_stride);
  const u32* B = reinterpret_cast<const u32*>(a.B + (long long)z * a.b_stride);
  AccI64 acc;
  int Kw;
  band_engine<SPLIT>(acc, A, a.L, B, a.L, K0, a.TI, smem, Kw);
  const int lane = threadIdx.x & 31;
  const int grp = lane / LPG, p = lane - grp * LPG;
  const int kmax = 2 * a.L - 1;
  if (grp == 0) {
    int64_t* dst = a.P + (long long)z * a.p_stride + Kw + 8 * p;
#pragma unroll
    for (int r = 0; r < 8; r++)
      if (Kw + 8 * p + r < kmax) dst[r] = acc.s[r];
  }
}

template <int SPLIT>
static cudaError_t launch_conv_t(const ConvArgs& a, cudaStream_t st) {
  const int grid = a.nprod * (a.nbands / 8);
  constexpr int CW = 8 * (32 / SPLIT);
  const size_t smem = (size_t)(2 * a.TI + 8 * CW) * sizeof(u32);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_conv<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_conv<SPLIT><<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_conv(const ConvArgs& a, cudaStream_t st) {
  switch (a.G) {
    case 1: return launch_conv_t<1>(a, st);
    case 2: return launch_conv_t<2>(a, st);
    case 4: return launch_conv_t<4>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace kmx
