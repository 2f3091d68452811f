/*
 * kmx.h -- C ABI of the B200-native multipoint Kronecker substitution path.
 *
 * The reference package (kronmul, pure Python) has no FFI; these entry points
 * are the batched native equivalents of its Python multiply entry points, and
 * are what a ctypes / cffi binding of the reference would bind:
 *
 *   kmx_ks_mul        <- kronmul.ksint.ks1_mul / ks2_mul / ks3_mul / ks4_mul
 *                        (pkg/src/kronmul/ksint.py:219-348), batched over pairs
 *   kmx_ks_mul_host   <- the same, host buffers in/out (the drop-in path)
 *   kmx_reconstruct   <- kronmul.ksint.reconstruct_overlapped
 *                        (pkg/src/kronmul/ksint.py:137-195)
 *   kmx_bks_mul       <- kronmul.bipoly.bks_standard / bks_reciprocal /
 *                        bks_negated / bks_four with ring_z()
 *                        (pkg/src/kronmul/bipoly.py:177-278)
 *   kmx_ks_params     <- kronmul.ksint.derive_params (ksint.py:82-98)
 *   kmx_mod_mul       <- kronmul.modpoly.mod_mul (modpoly.py:95-115), batched
 *   kmx_bks_mod_mul   <- kronmul.bipoly.bks_* with ring_zmod(n) (bipoly.py:59-72, :177-278)
 *
 * Conventions
 *   - Plain pointers and sizes; no torch types.  Device entry points take
 *     device pointers and a cudaStream_t passed as void*; they are
 *     stream-ordered and asynchronous.  Device-side consistency errors
 *     (ReconstructionError, inexact halving/shift, coefficient out of range)
 *     are latched in a flag inside the caller-owned workspace; read it with
 *     kmx_ws_status() (synchronises the stream).
 *   - Coefficients are little-endian 32-bit words: f is [batch][len_f][in_words],
 *     g is [batch][len_g][in_words], h is [batch][len_f+len_g-1][out_words]
 *     with out_words >= kmx_ks_out_words(...).
 *   - Variant numbering follows the reference names (ksint.py:8-12):
 *     1 = standard (2^N), 2 = reciprocal (2^N, 2^-N), 3 = negated (+-2^N),
 *     4 = four-point (+-2^N, +-2^-N).
 *   - KMX_SIGNED: coefficients are two's-complement coeff_bits-bit integers
 *     (coeff_bits <= 32, in_words == 1); the product coefficients are written
 *     in two's complement.  The reference rejects negative coefficients
 *     (pack.py:44-46); the signed path is the bias lift of SURVEY.md §8(c).
 *
 * Return codes map to the reference's exceptions:
 *   KMX_OK 0; KMX_EINVAL -1 -> ValueError (pack.py:39-59, ksint.py:84-87);
 *   KMX_ERECON -2 -> ReconstructionError (ksint.py:44-45, :157-177);
 *   KMX_EINEXACT -3 -> ValueError (bignat.py:265-269, :310-317, :446-447);
 *   KMX_ECUDA -4; KMX_ENOMEM -5.
 */
#ifndef KMX_H
#define KMX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KMX_OK 0
#define KMX_EINVAL (-1)
#define KMX_ERECON (-2)
#define KMX_EINEXACT (-3)
#define KMX_ECUDA (-4)
#define KMX_ENOMEM (-5)

/* flags */
#define KMX_SIGNED 1u          /* two's-complement input coefficients        */
#define KMX_NO_VALIDATE 2u     /* skip the 0 <= c < 2^b range check           */
#define KMX_NO_SPLIT 4u        /* kmx_ks_mul: do not split the batch over two streams */
#define KMX_NO_TUNE 8u         /* kmx_ks_mul: no first-call timing runs (model-chosen plan, default schedule) */

/* Derived parameters (ksint.py:82-98).  out[0..7] = e, N1, N2, N4,
 * four_point_safe, out_len, limbs of the packed f operand, limbs of the
 * packed g operand for `variant` (after any KS4 -> KS1 fallback). */
int kmx_ks_params(int variant, int len_f, int len_g, int coeff_bits, unsigned flags,
                  int64_t* out8);

/* Minimum out_words for h: ceil(N1 / 32) (the reference's out_bound_bits =
 * 2b+e, ksint.py:74-79). */
int kmx_ks_out_words(int len_f, int len_g, int coeff_bits, unsigned flags);

/* Bytes of device workspace needed by kmx_ks_mul for this problem. */
size_t kmx_ks_workspace_bytes(int variant, int batch, int len_f, int len_g, int coeff_bits,
                              unsigned flags);

/* Batched KS product on the device (asynchronous on `stream`).
 *
 * First call per (device, shape, batch) with batch >= 64, outside a CUDA
 * graph capture and without KMX_NO_TUNE: the call measures its batch-split
 * schedule and tensor-core tiling by running the product several times on
 * `stream` and BLOCKS the host until those timing runs finish (each run
 * writes the same bit-exact h).  The choice is cached per device; later calls
 * (and graph captures) are asynchronous.  Pass KMX_NO_TUNE (or set
 * KMX_TC_AUTOTUNE=0 and KMX_SPLIT) for a strictly asynchronous first call. */
int kmx_ks_mul(int variant, int batch, int len_f, int len_g, int coeff_bits,
               const uint32_t* f, const uint32_t* g, int in_words,
               uint32_t* h, int out_words,
               void* workspace, size_t ws_bytes, unsigned flags, void* stream);

/* Read and clear the workspace's latched device error (synchronises stream). */
int kmx_ws_status(void* workspace, void* stream);

/* Per-operand statistics of the last kmx_ks_mul on this workspace
 * (synchronises stream): the reference's MulStats.limb_products under
 * classical multiplication, i.e. the sum over sub-products of
 * limbs64(x) * limbs64(y) on the normalized packed operands
 * (bignat.py:327-330).  Written to *limb_products64 as a batch total. */
int kmx_ws_limb_products(void* workspace, int variant, int batch, int len_f, int len_g,
                         int coeff_bits, unsigned flags, uint64_t* limb_products64,
                         void* stream);

/* Host-buffer entry point: copies f, g to the device, runs kmx_ks_mul,
 * copies h back and checks the device error flag.  Thread-safe (per-device
 * cached buffers under a mutex).  Pinned host memory gives full PCIe speed. */
int kmx_ks_mul_host(int variant, int batch, int len_f, int len_g, int coeff_bits,
                    const uint32_t* f, const uint32_t* g, int in_words,
                    uint32_t* h, int out_words, unsigned flags,
                    uint64_t* limb_products64 /* nullable: MulStats count */);

/* K1 alone: kronmul.pack.pack (kind 0), pack_negated (1), pack_reversed (2),
 * pack_negated_reversed (3) (pack.py:79-110) of `batch` coefficient vectors
 * [batch][len][in_words] at width_bits (2*width_bits >= coeff_bits, else
 * KMX_EINVAL as pack.py:55-59).  out: [batch][out_limbs] |value| little-endian
 * limbs, out_limbs >= kmx_pack_limbs() and a multiple of 4 (out 16-byte
 * aligned: K1 stores limb quads); meta (required on the device entry,
 * nullable on the host entry):
 * [batch][2] = {sign (1: negative), bit length of |value|}.  Coefficients
 * outside [0, 2^coeff_bits) latch KMX_EINVAL (read with kmx_ws_status);
 * the device workspace is >= 256 bytes. */
int kmx_pack_limbs(int len, int width_bits, int coeff_bits);
int kmx_pack(int kind, int batch, int len, int width_bits, int coeff_bits, const uint32_t* coeffs, int in_words,
             uint32_t* out, int out_limbs, uint32_t* meta, void* workspace, size_t ws_bytes, void* stream);
int kmx_pack_host(int kind, int batch, int len, int width_bits, int coeff_bits, const uint32_t* coeffs,
                  int in_words, uint32_t* out, int out_limbs, uint32_t* meta);

/* Overlap reconstruction of `batch` independent digit-stream pairs on the
 * device: fwd, rev are [batch][count+1][dwords] (rev listed most significant
 * first, ksint.py:101-109), width_bits <= 32*dwords; h is
 * [batch][count][hwords] with hwords >= ceil(2*width_bits/32).  carries
 * (nullable) receives [batch][2*count+1] bytes: the count+1 forward-stream
 * carries then the count reverse-stream carries (ksint.py:182-195,
 * with_carries=True). */
size_t kmx_reconstruct_workspace_bytes(int batch, int count, int dwords);
int kmx_reconstruct(int batch, int count, int width_bits, const uint32_t* fwd,
                    const uint32_t* rev, int dwords, uint32_t* h, int hwords,
                    void* workspace, size_t ws_bytes, uint8_t* carries, void* stream);
int kmx_reconstruct_host(int batch, int count, int width_bits, const uint32_t* fwd,
                         const uint32_t* rev, int dwords, uint32_t* h, int hwords,
                         uint8_t* carries);

/* Bivariate R[x,y] -> R[x] reductions over R = Z.  f, g: [batch][lx][ly]
 * int32 (coeffs[i][j] of x^i y^j, bipoly.py:75-97); h: [batch][2lx-1][2ly-1]
 * int64.  coeff_bits bounds |c| < 2^coeff_bits (<= 30) and must keep every
 * univariate product coefficient inside int64 (checked -> KMX_EINVAL). */
size_t kmx_bks_workspace_bytes(int variant, int batch, int lx, int ly);
/* Workspace for this coefficient bound: large enough for the univariate
 * products to run on the integer KS path (tensor cores) where that is the
 * engine; kmx_bks_workspace_bytes() sizes the k_conv engine, which
 * kmx_bks_mul falls back to when the workspace is smaller. */
size_t kmx_bks_workspace_bytes_cb(int variant, int batch, int lx, int ly, int coeff_bits);
/* Engine of the univariate products for this shape: 0 = the int32 x int32 ->
 * int64 IMAD convolution (k_conv), 1..4 = the integer KS path with that
 * variant (tensor cores). */
int kmx_bks_uni_engine(int variant, int lx, int ly, int coeff_bits);
int kmx_bks_mul(int variant, int batch, int lx, int ly, int coeff_bits,
                const int32_t* f, const int32_t* g, int64_t* h,
                void* workspace, size_t ws_bytes, void* stream);
int kmx_bks_mul_host(int variant, int batch, int lx, int ly, int coeff_bits,
                     const int32_t* f, const int32_t* g, int64_t* h);

/* Bivariate reductions over R = Z for coefficients of any width (bipoly.py
 * :177-278 with ring_z(); the reference takes any integer): f, g
 * [batch][lx][ly][in_words] two's-complement integers with |c| < 2^coeff_bits
 * (checked -> KMX_EINVAL via kmx_ws_status); h [batch][2lx-1][2ly-1]
 * [out_words] two's complement, out_words >= kmx_bks_wide_out_words().  The
 * reduction runs over Z/p_i for word-sized primes (kmx_bks_mod_mul each) and
 * the coefficients are recovered by CRT on the device. */
int kmx_bks_wide_out_words(int lx, int ly, int coeff_bits);
size_t kmx_bks_wide_workspace_bytes(int variant, int batch, int lx, int ly, int coeff_bits);
int kmx_bks_wide_mul(int variant, int batch, int lx, int ly, int coeff_bits, const uint32_t* f, const uint32_t* g,
                     int in_words, uint32_t* h, int out_words, void* workspace, size_t ws_bytes, void* stream);
int kmx_bks_wide_mul_host(int variant, int batch, int lx, int ly, int coeff_bits, const uint32_t* f,
                          const uint32_t* g, int in_words, uint32_t* h, int out_words);

/* (Z/nZ)[x] products, 2 <= n < 2^64 (kronmul.modpoly.mod_mul,
 * modpoly.py:95-115): f [batch][len_f], g [batch][len_g] u64 coefficients in
 * [0, n) (checked -> KMX_EINVAL, modpoly.py:47-58); h [batch][len_f+len_g-1]
 * u64 = the coefficients of f*g reduced mod n.  The lift uses b =
 * max(1, bitlen(n-1)) (modpoly.py:104) and KS variant 1..4 (AUTO is resolved
 * by the caller, modpoly.py:105-106). */
size_t kmx_mod_workspace_bytes(int variant, int batch, int len_f, int len_g, uint64_t modulus);
int kmx_mod_mul(int variant, int batch, int len_f, int len_g, uint64_t modulus,
                const uint64_t* f, const uint64_t* g, uint64_t* h,
                void* workspace, size_t ws_bytes, void* stream);
int kmx_mod_mul_host(int variant, int batch, int len_f, int len_g, uint64_t modulus,
                     const uint64_t* f, const uint64_t* g, uint64_t* h,
                     uint64_t* limb_products64 /* nullable: MulStats count */);

/* Bivariate R[x,y] -> R[x] reductions over R = Z/nZ, 2 <= n < 2^64
 * (bipoly.py:177-278 with ring_zmod(n), :59-72).  f, g: [batch][lx][ly] u64
 * residues in [0, n) (checked -> KMX_EINVAL); h: [batch][2lx-1][2ly-1] u64.
 * The univariate products run through kmx_mod_mul.  Variants 3 and 4 need
 * the ring's halving and return KMX_EINVAL for even n (the reference raises
 * MissingHalveError, bipoly.py:116-118). */
size_t kmx_bks_mod_workspace_bytes(int variant, int batch, int lx, int ly, uint64_t modulus);
int kmx_bks_mod_mul(int variant, int batch, int lx, int ly, uint64_t modulus,
                    const uint64_t* f, const uint64_t* g, uint64_t* h,
                    void* workspace, size_t ws_bytes, void* stream);
int kmx_bks_mod_mul_host(int variant, int batch, int lx, int ly, uint64_t modulus,
                         const uint64_t* f, const uint64_t* g, uint64_t* h);

/* Measured IMAD.WIDE.U32 throughput on device 0 (32x32->64 products per
 * second, full chip), the roofline denominator for the multiply kernels. */
double kmx_imad_peak(int iters);

/* Engine the multiply stage (K2) uses for this product shape: 0 = the
 * integer-pipe schoolbook (IMAD.WIDE.U32, kmx_mul.cu), 1 = the tcgen05 u8
 * byte convolution with TMEM accumulators (kmx_tc.cu).  KMX_TC=0 in the
 * environment forces 0.  Negative: error code. */
int kmx_mul_engine(int variant, int len_f, int len_g, int coeff_bits, unsigned flags);

/* Karatsuba levels (bignat.py:344-371) the multiply stage applies above the
 * engines for this shape (0: one engine launch per product). */
int kmx_mul_karatsuba_levels(int variant, int batch, int len_f, int len_g, int coeff_bits, unsigned flags);

/* The multiply plan a kmx_ks_mul of this shape runs with (split schedules
 * aside: for `batch` products per launch): out8 = {engine (0 integer pipe,
 * 1 tiled tensor-core kernel, 2 chunked single-tile kernel, 3 Karatsuba levels
 * over the engines with out8[1] = levels, 4 swizzled-window tensor-core
 * kernel, 5 its M = 64 two-window form), H (MMA N = 16 H), NW, KC (K-steps
 * per stage / chunk), tiles per CTA, MMAs per product, shared-memory operand
 * bytes per product, issued byte MACs per product}; fields 1-7 are filled
 * for engines 1, 4 and 5. */
int kmx_mul_plan(int variant, int batch, int len_f, int len_g, int coeff_bits, unsigned flags, int64_t* out8);

/* Measured dense u8 x u8 -> s32 tcgen05.mma throughput on the current
 * device (multiply-accumulates per second, M=128 N=256 K=32 from shared
 * memory, all SMs): the tensor roofline denominator for K2. */
double kmx_tc_peak(int iters);

/* The same microbenchmark for M=128 and N in {16, 32, 48, 64, 96, 128, 256}:
 * the SS-mode rate at the tile widths K2 issues (each MMA re-reads its 4 KB A
 * tile from shared memory), i.e. K2's same-shape ceiling. */
double kmx_tc_peak_n(int n, int iters);

/* Human-readable message for a return code. */
const char* kmx_error_string(int code);

/* Number of kernels launched by the last kmx_ks_mul / kmx_bks_mul call on
 * this thread (for the bench's gpu_launches count). */
int kmx_last_launch_count(void);

/* Per-kernel CUDA-event timing of kmx_ks_mul on the calling thread (events
 * recorded on the caller's stream around each launch).  kmx_prof_read
 * synchronises on the last call's events and writes the durations in ms to
 * ms[0..5] = pack, multiply, finish, reconstruct, bias, mod reduction (0 if
 * not launched; for kmx_bks_mul: 0 evaluation, 1 convolution, 2 recovery);
 * returns the number of kernels timed. */
void kmx_prof_enable(int on);
int kmx_prof_read(float* ms, int nslots);

#ifdef __cplusplus
}
#endif
#endif /* KMX_H */
