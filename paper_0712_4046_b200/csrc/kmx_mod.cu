// kmx_mod.cu -- the (Z/nZ)[x] front end (kronmul.modpoly.mod_mul,
// modpoly.py:95-115): the lifted product comes out of the KS path as
// [pair][k][ow] little-endian words (< 2^(2b+e), b = bitlen(n-1)); K9
// reduces every coefficient mod n (modpoly.py:115, `c % n`) into one u64.
//
// Reduction: v = sum_i w_i 2^(32 i) with ow <= 8 words; with the host's
// t_i = 2^(32 i) mod n, acc = sum_i w_i t_i < 8 * 2^96 fits 128 bits and
// v == acc (mod n); one 128-by-64 remainder finishes.  The same grid checks
// the ModPoly invariant 0 <= c < n of the inputs (modpoly.py:47-58) and
// latches ERR_INVAL (-> ValueError) on a violation.
#include "kmx_common.cuh"
#include "kmx_internal.h"

namespace kmx {

__global__ void __launch_bounds__(256) k_modred(ModRedArgs a) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.count; i += stride) {
    const u32* w = a.prod + i * a.ow;
    unsigned __int128 acc = 0;
#pragma unroll 4
    for (int q = 0; q < a.ow; q++) acc += (unsigned __int128)__ldg(w + q) * a.tpow[q];
    a.out[i] = (u64)(acc % a.n);
    if (i < a.nf && __ldg(a.f + i) >= a.n) raise_err(a.err, ERR_INVAL);
    if (i < a.ng && __ldg(a.g + i) >= a.n) raise_err(a.err, ERR_INVAL);
  }
}

cudaError_t launch_modred(const ModRedArgs& a, cudaStream_t st) {
  long long blocks = (a.count + 255) / 256;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  if (blocks < 1) blocks = 1;
  k_modred<<<(int)blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace kmx
