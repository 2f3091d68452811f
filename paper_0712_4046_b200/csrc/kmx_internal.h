// Internal launch interface between the C-ABI layer (kmx_api.cu) and the
// kernels (kmx_ks.cu, kmx_bivar.cu).  Host-visible structs only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kmx {

// ------------------------------------------------------------------ pack
// One packed operand family: the value of a coefficient vector at +-2^N or
// +-2^-N (pack.py:79-110).  kind: 0 = pack, 1 = pack_negated,
// 2 = pack_reversed, 3 = pack_negated_reversed.
struct PackOp {
  const uint32_t* coeffs;     // pair 0's coefficients; pair p at + p*coeff_pair_stride
  long long coeff_pair_stride;
  int len;
  int kind;
  uint32_t* out;              // pair 0's operand; pair p at + p*out_pair_stride
  long long out_pair_stride;
  uint32_t* meta;             // pair 0's [sign, bitlen]; pair p at + p*meta_pair_stride
  long long meta_pair_stride;
  int m;                      // limbs of this operand
  int validate;               // check 0 <= c < 2^b on this operand's coefficients
  unsigned long long* prefix; // signed path: prefix sums of the lifted coefficients (or null)
  long long prefix_pair_stride;
};
struct PackArgs {
  PackOp op[8];
  int nops;
  int N;                      // evaluation width (bits)
  int b;                      // coefficient bound (bits)
  int in_words;
  int bias;                   // signed inputs: add 2^(b-1) (bias lift)
  uint32_t* err;
  int stage;                  // set by launch_pack: coefficients staged in shared memory
  int fast1;                  // set by launch_pack: loop-free bitstream windows allowed (KMX_PACK_FAST)
  void* scratch;              // segmented pack (kmx_packseg.cu): orders and segment carry maps
  size_t scratch_bytes;
};
size_t pack_seg_scratch_bytes(int batch, int nops, int mmax);

// -------------------------------------------------------------- multiply
// G carries the row-split factor SPLIT (1, 2, 4): bands are CW = 256/SPLIT
// columns wide, 8 bands per CTA; TI is the number of operand rows staged
// per shared-memory chunk (TR).
struct MulArgs {
  const uint32_t* A; long long a_stride; int ma;  // product z: A + z*a_stride
  const uint32_t* B; long long b_stride; int mb;
  uint32_t* P; long long p_stride;                // digits, p_stride >= nbands*CW
  unsigned long long* spill;                      // [z][nbands][2]
  int nprod, nbands, G, TI;
  int* counter;                                   // work-unit counter, zeroed before launch
  int flags_no_tune;                              // KMX_NO_TUNE: the cost model's tiling, no timing runs
  uint32_t* err;                                  // error flag (Karatsuba recombination check)
};
struct ConvArgs {
  const int32_t* A; long long a_stride;
  const int32_t* B; long long b_stride;
  int L;                                          // operand length (both)
  int64_t* P; long long p_stride;                 // 2L-1 int64 column sums
  int nprod, nbands, G, TI;
  int* counter;                                   // work-unit counter, zeroed before launch
};
void mul_geometry(int ma, int mb, int* split, int* cw, int* nbands, int* tr);
// K1 staging limits (kmx_pack.cuh PK_PAD / PK_STAGE_WORDS), visible to the host
constexpr int PK_PAD_WORDS = 64;
constexpr int PK_STAGE_LIMIT_WORDS = 12288;
// K2 on tcgen05 (kmx_tc.cu): same MulArgs contract, zero band spills.
bool tc_supported(int ma, int mb, size_t stage_bytes = 0);
// pk != nullptr: fused pack -- each product's CTA packs its two operands
// (pack ops s and P + s of its pair) straight into shared memory; the packed
// operands never reach global memory (MulArgs A/B unused).
cudaError_t launch_tcmul(const MulArgs& a, cudaStream_t st, const PackArgs* pk = nullptr, int P = 1);
// K2 with swizzled sliding windows and a phase table (kmx_tcs.cu): same
// MulArgs contract; pitch = 32 / 64 / 128 (= the MMA's N).
struct TcsPlan {
  int pitch, KS, ntiles;
  int persist, NS;  // the persistent warp-specialized form and its operand stages
  int nch;          // accumulation chains per tile (2 past 64 KB of the shorter operand)
  size_t smem;
  long long mmas;  // MMAs per product
  double cost;     // modelled SM cycles per product
};
bool tcs_plan(int ma, int mb, int pitch, int persist, TcsPlan& p);
struct FinishArgs;
// fin != nullptr: one CTA per pair multiplies the pair's products and runs the
// warp-per-stream finish (K3) for it (single-tile plans only)
cudaError_t launch_tcs(const MulArgs& a, const TcsPlan& p, cudaStream_t st, const FinishArgs* fin = nullptr);
bool launch_tcmul_finish(const MulArgs& a, const FinishArgs& fa, int batch, cudaStream_t st, cudaError_t* err);
double measure_tc_peak(int iters);
double measure_tc_peak_shape(int n, int iters);
// engine choice (kmx_api.cu): the tensor cores for this shape, and whether
// some engine takes the whole product (else Karatsuba splits it)
bool mul_use_tensor(int ma, int mb);
bool mul_engine_takes(int ma, int mb);

// ---------------------------------------------------- Karatsuba (kmx_kara.cu)
// Linear-combination normalizer: out[z] = sum_t sign_t term_t[z] 2^(32 off_t),
// each term a product in the engines' format (limbs + optional band spills).
constexpr int LC_MAXT = 5;
constexpr int KARA_MAX_DEPTH = 4;
struct LcTerm {
  const uint32_t* p; long long stride; long long len; long long off; int sign;
  const unsigned long long* spill; int nbands;    // band spills, band bi at spill[z * spill_stride + 2 bi]
  long long spill_stride;                         // u64 entries per z (0: nbands * 2)
  const uint32_t* smeta; long long smeta_stride; int smeta_off;  // optional: sign *= -1 when
                                                  // smeta[z*stride] ^ smeta[z*stride + off] (mul_signed)
};
struct LcArgs {
  LcTerm t[LC_MAXT];
  int nt;
  uint32_t* out; long long out_stride; long long out_len;
  int nchunks;                                    // set by launch_lincomb
  void* maps;                                     // [nprod][nchunks] chunk carry maps
  uint32_t* err;
};
cudaError_t launch_lincomb(const LcArgs& a, long long nprod, cudaStream_t st);
size_t lc_map_bytes(long long nprod, int out_len);
bool kara_used(int ma, int mb);
int kara_levels(int ma, int mb);
size_t kara_ws_bytes(int ma, int mb, long long nprod);
cudaError_t launch_kara(const MulArgs& a, void* ws, cudaStream_t st, int* nlaunch);



// Signed inputs (bias lift): the coefficient writers apply
// h = h' - 2^(b-1) (J*f' + J*g') + 2^(2b-2) (J*J) before storing, from the
// prefix sums PF, PG of the lifted inputs ([pair][lf+1 | lg+1]).
struct BiasFix {
  const unsigned long long* pf;
  long long pair_stride;
  int lf, lg, b, enabled;
  int lgpad;                  // staged (padded) copy: entry i at i + (i >> lgpad); -1: unpadded
};

// ---------------------------------------------------------------- finish
// One output digit stream of one pair: digits of (P + qsign*sgn(Q)*|Q|) >> off
// at width W (the half-sum / half-difference and the exact shifts of
// ksint.py:270-273 and :320-335, and the unpacks of _unpack_ints).
struct Stream {
  int zP, zQ;                 // product slots inside a pair
  int qsign;                  // 0: P alone; +1 / -1: P + / - signed Q
  int qmeta;                  // operand-meta slot index (f side) of Q's first operand
  long long off;              // first bit of digit 0
  int W;                      // digit width in bits
  int cnt;                    // number of digits (all higher bits must be zero)
  int mode;                   // 0: coefficient output, 1: digit buffer
  int pos0, pstride;          // mode 0: h[pair][pos0 + j*pstride]
  int dslot;                  // mode 1: digit-buffer slot inside the pair
  int reversed;               // mode 1: store digit j at index cnt-1-j
};
struct FinishArgs {
  Stream s[4];
  int ns;
  const uint32_t* P; long long p_stride; int mp; int nprod_pair;
  const unsigned long long* spill; int nbands; int band_cols;
  const uint32_t* meta; int meta_per_pair;        // 2 words per operand
  int mf_slot_stride;                             // operand meta: f ops at [sub], g ops at [P+sub]
  uint32_t* h; int out_words; long long h_pair_stride;
  uint32_t* dbuf; int dwords; long long dslot_stride; int dslots_pair;
  BiasFix bias;
  uint32_t* err;
  uint8_t* cmaps; int nchunks;                    // chunk-parallel finish: [pair*ns + si][nchunks] carry maps
};
constexpr int FIN_THREADS = 256;
constexpr int FIN_HALO = 32;
// warp-per-stream finish (kmx_finish.cu) for short streams / many streams
bool finish_use_warp(const FinishArgs& a, int batch);
bool finish_use_chunks(const FinishArgs& a, int batch);
cudaError_t launch_finish_w(const FinishArgs& a, int batch, cudaStream_t st);

// --------------------------------------------------------- reconstruction
struct ReconStream { int fslot, rslot, count, pos0, pstride; };
struct ReconArgs {
  ReconStream s[2];
  int ns;
  int batch;
  int W;
  const uint32_t* dbuf; int dwords; long long dslot_stride; int dslots_pair;
  uint32_t* h; int out_words; long long h_pair_stride;
  uint8_t* carries;           // optional [batch*ns][2*count+1]: fwd carries, rev carries
  BiasFix bias;
  uint32_t* err;
  int rch;                    // steps per staged chunk (set by launch_recon)
  int sequential;             // force the one-thread-per-stream kernel
  int stage;                  // k_recon_par: stream digits staged in shared memory
  uint32_t* diag;             // optional counter of sequential fallbacks
  int rw_slice;               // k_recon_warp: shared-memory words per warp
  int bias_smem;              // k_recon_par: stage the signed path's prefix sums in shared memory
  int spec;                   // k_recon_par: speculative stores from this scan round on (0: never)
};

// ---------------------------------------------------------- signed (bias)
struct BiasArgs {
  const uint32_t* f; const uint32_t* g; int lf, lg, b;
  uint32_t* h; int out_words;
  unsigned long long* scratch;  // [batch][lf+lg+2]
  int batch;
};

// per-kernel CUDA-event timing (kmx_prof_*): slots 0 pack / beval, 1 mul / conv,
// 2 finish / brecover, 3 recon, 4 bias, 5 modred
void prof_mark(int slot, bool begin, cudaStream_t st);
void prof_reset();
// nested C-ABI calls (the bivariate path's KS products) keep the caller's slots
bool prof_suspend();
void prof_keep(int slot);
void prof_resume(bool was);

// ------------------------------------------------------------- (Z/nZ)[x]
// K9: h[i] = (sum_q prod[i][q] 2^(32q)) mod n, tpow[q] = 2^(32q) mod n
struct ModRedArgs {
  const uint32_t* prod; int ow; long long count;
  unsigned long long n; unsigned long long tpow[8];
  unsigned long long* out;
  const unsigned long long* f; long long nf;   // inputs: 0 <= c < n check
  const unsigned long long* g; long long ng;
  uint32_t* err;
};
cudaError_t launch_modred(const ModRedArgs& a, cudaStream_t st);

// kernels launched by the last C-ABI call on this thread (bench gpu_launches)
extern thread_local int g_launches;

// launchers (return cudaError_t of the launch)
cudaError_t launch_pack(const PackArgs& a, int batch, cudaStream_t st);
cudaError_t launch_mul(const MulArgs& a, cudaStream_t st);
cudaError_t launch_conv(const ConvArgs& a, cudaStream_t st);
cudaError_t launch_finish(const FinishArgs& a, int batch, cudaStream_t st);
cudaError_t launch_recon(const ReconArgs& a, cudaStream_t st);
// K4 with one CTA per pair for digits of at most 64 bits (kmx_recon2.cu)
bool recon_pair_ok(const ReconArgs& a);
cudaError_t launch_recon_pair(const ReconArgs& a, cudaStream_t st);
// K3 + K4 fused for ks2 / ks4 when both apply (warp finish, staged
// reconstruction); *used = false: nothing launched, run them separately
cudaError_t launch_finrec(const FinishArgs& fa, const ReconArgs& ra, int batch, cudaStream_t st, bool* used);
cudaError_t launch_bias(const BiasArgs& a, cudaStream_t st);
double measure_imad_peak(int iters);

// ---------------------------------------------------------------- bivariate
struct BivarPlan {
  int variant, lx, ly, batch;
  int P;          // univariate products per pair
  int Lu;         // univariate operand length
  int spacing;    // chunk spacing in the evaluation
  int n4;         // four-point half length
  int cbits;      // declared bound |c| < 2^cbits, checked on the device (ERR_INVAL)
  int uni;        // univariate products: 0 = k_conv (IMAD), 1..4 = the integer KS path (variant)
  int ebits;      // signed width of the evaluations (two's complement) for the KS path
};
cudaError_t launch_bivar(const BivarPlan& p, const int32_t* f, const int32_t* g, int64_t* h,
                         int32_t* evals, int64_t* prods, uint32_t* err, cudaStream_t st,
                         int* nlaunch, void* ks_ws, size_t ks_ws_bytes, uint32_t* err0);

// ------------------------------------------- wide digits (kmx_wide.cu)
// Digit widths past the chunked finish / register reconstruction
// (W > 32 (FIN_HALO - 1) or reconstruction digits > 17 words): the
// numerator of each stream normalized by the linear-combination kernels, a
// bit-field gather for the digits, a sequential multiword reconstruction.
struct WideDigitArgs {
  const uint32_t* T; long long t_stride; long long t_len;  // normalized numerator [pair][t_len]
  Stream s;
  uint32_t* h; int out_words; long long h_pair_stride;
  uint32_t* dbuf; int dwords; long long dslot_stride; int dslots_pair;
  uint32_t* err;
  int batch;
};
cudaError_t launch_wide_digits(const WideDigitArgs& a, cudaStream_t st);
size_t wide_recon_scratch_words(int batch, int ns, int dwords);
// ReconArgs with any dwords; scratch: wide_recon_scratch_words(...) words
cudaError_t launch_wide_recon(const ReconArgs& a, uint32_t* scratch, cudaStream_t st);

}  // namespace kmx
