// tcgen05.mma kind::i8 throughput microbenchmark (SS mode, M = 128).
//
// Each CTA issues back-to-back u8 x u8 -> s32 MMAs from shared memory into
// one TMEM accumulator and commits every 32 instructions.  Reports int8
// MAC/s for N in {16, 32, 64, 128, 256}, with A either a standard packed
// K-major tile (LBO = 128, SBO = 256... per 8-row group) or the sliding
// layout kmx_tc.cu uses (LBO = 16, SBO = 128 over a raw byte string).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_peak tc_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <int N, int SLIDE, int SBOA = 128>
__global__ void __launch_bounds__(128) k_peak(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) unsigned long long mbar;
  constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  constexpr int KS = 8;  // K-steps resident (A: 8 x 4 KB, B: 8 x N*32)
  constexpr int ABYTES = (SBOA * 16 > 8 * 4096 ? SBOA * 16 : 8 * 4096) + 4096;
  unsigned char* A = sm;
  unsigned char* B = sm + ABYTES;
  for (int i = threadIdx.x; i < (ABYTES + KS * N * 32) / 4; i += 128)
    reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    for (int it = 0; it < iters; it++) {
      for (int k = 0; k < 32; k++) {
        const int s = k % KS;
        uint64_t ad = SLIDE ? sdesc(smem_u32(A) + 32 * s, 16, SBOA)
                            : sdesc(smem_u32(A) + 4096 * s, 128, 256);
        uint64_t bd = sdesc(smem_u32(B) + N * 32 * s, 128, 256);
        uint32_t acc = (it | k) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(tm), "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
      uint32_t done = 0;
      do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}\n"
                     : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
      } while (!done);
      phase ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u) sink[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
  }
}

template <int N, int SLIDE, int SBOA = 128>
double run(int ctas_per_sm, int iters) {
  const size_t smem = (SBOA * 16 > 8 * 4096 ? SBOA * 16 : 8 * 4096) + 4096 + 8 * N * 32 + 1024;
  cudaFuncSetAttribute(k_peak<N, SLIDE, SBOA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * ctas_per_sm;
  k_peak<N, SLIDE, SBOA><<<grid, 128, smem>>>(2, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_peak<N, SLIDE, SBOA><<<grid, 128, smem>>>(iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  cudaFree(sink);
  const double macs = (double)grid * iters * 32 * 128.0 * N * 32;
  return macs / (ms * 1e-3);
}

int main() {
  const int iters = 2000;
  printf("{\"unit\": \"int8 MAC/s\", \"M\": 128, \"K_per_mma\": 32, \"results\": [\n");
#define R(N, S, C)                                                                                            \
  printf("  {\"N\": %d, \"sliding_A\": %d, \"ctas_per_sm\": %d, \"mac_per_s\": %.4e},\n", N, S, C, run<N, S>(C, iters));
  R(16, 0, 2) R(16, 1, 2) R(16, 1, 4) R(32, 0, 2) R(32, 1, 2) R(64, 0, 2) R(64, 1, 2) R(128, 0, 2) R(128, 1, 2)
  R(256, 0, 1) R(256, 1, 1)
#define RS(N, SB, C)                                                                                            \
  printf("  {\"N\": %d, \"sliding_A\": 1, \"sbo_a\": %d, \"ctas_per_sm\": %d, \"mac_per_s\": %.4e},\n", N, SB, C, run<N, 1, SB>(C, iters));
  RS(32, 256, 2) RS(32, 272, 2) RS(64, 512, 2) RS(64, 528, 2) RS(64, 1024, 2) RS(128, 1024, 2) RS(128, 1040, 2) RS(128, 2048, 1)
  printf("  {}\n]}\n");
  return 0;
}
