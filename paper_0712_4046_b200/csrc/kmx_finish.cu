// kmx_finish.cu -- K3 for short streams: one WARP per output digit stream
// (the same contract as k_finish in kmx_ks.cu: half-sum / half-difference
// P + s*Q with the band spills folded in, exact halving and shifts,
// W-bit digit extraction and the ERR_INEXACT checks; ksint.py:219-279,
// :305-345; bignat.py:265-274, :310-317, :431-450).
//
// Why a warp: at the BASELINE shapes a stream is a few hundred to a few
// thousand limbs (c2 ks4: 1218), so a 256-thread block with 2048-limb chunks
// idles most of its lanes and pays a block barrier per scan.  Here a warp
// walks its stream in 256-limb chunks (8 limbs per lane) with shuffles only,
// and the carry resolution is cheap:
//   * y_v = P_v + s Q_v (+ spill) is split y = lo + 2^32 hi and hi moved one
//     limb up (z_v = lo_v + hi_(v-1)), so every carry lies in {-1, 0, 1};
//   * each lane resolves its 8 limbs sequentially assuming carry-in 0, which
//     gives its carry-out c0 and digits D; a carry-in of +1 (-1) changes the
//     carry-out only if D is all ones (all zeros), so the lane's carry map is
//     (c0 - all0, c0, c0 + allF) -- three compares instead of a map per limb;
//   * one 5-step shuffle scan composes the lane maps; the lanes whose
//     carry-in is nonzero ripple it through their 8 digits.
// The normalized limbs go to a per-warp shared buffer (with a 32-word halo
// for digits straddling chunks) and the lanes extract digits from it.
#include <cstdlib>

#include "kmx_common.cuh"
#include "kmx_internal.h"
#include "kmx_finish.cuh"

namespace kmx {

namespace {

__global__ void __launch_bounds__(32 * FW_WARPS, 8) k_finish_w(FinishArgs a, long long nstreams) {
  __shared__ __align__(16) u32 sbuf[FW_WARPS][FIN_HALO + FW_CH];
  const int wid = threadIdx.x >> 5;
  const long long gs = (long long)blockIdx.x * FW_WARPS + wid;
  if (gs >= nstreams) return;  // warp-uniform
  const int pair = (int)(gs / a.ns);
  const int si = (int)(gs - (long long)pair * a.ns);
  finish_warp_stream(a, pair, si, sbuf[wid], GlobalDigitSink{&a});
}

}  // namespace

// Warp-per-stream finish when streams are short (few chunks each) or there
// are enough of them to fill the chip with warps; KMX_FINISH_WARP=0/1 forces.
bool finish_use_warp(const FinishArgs& a, int batch) {
  static const int force = getenv("KMX_FINISH_WARP") ? atoi(getenv("KMX_FINISH_WARP")) : -1;
  if (force >= 0) return force != 0;
  const long long streams = (long long)batch * a.ns;
  return a.mp <= 1024 || (a.mp <= 8192 && streams >= 148LL * 8);
}

cudaError_t launch_finish_w(const FinishArgs& a, int batch, cudaStream_t st) {
  const long long ns = (long long)batch * a.ns;
  const long long blocks = (ns + FW_WARPS - 1) / FW_WARPS;
  k_finish_w<<<(unsigned)blocks, 32 * FW_WARPS, 0, st>>>(a, ns);
  return cudaGetLastError();
}

}  // namespace kmx
