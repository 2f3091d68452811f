// tcgen05.mma kind::i8 with the A operand in TENSOR MEMORY (M = 128):
// layout check and throughput.
//
// 1. layout: every lane writes its row's 32 bytes with tcgen05.st.32x32b.x8
//    (word c of lane m = A[m][4c..4c+3], little-endian), B is a K-major
//    SWIZZLE_NONE smem tile; D = A B^T is compared with the host result.
// 2. throughput: back-to-back MMAs from a ring of TMEM A stages, B in smem,
//    for N in {16..256}; then the same with four warps re-writing the A
//    stages through an mbarrier ring (the producer pattern a kernel would use).
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_ts tc_ts.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d), "r"(a), "l"(bd), "r"(idesc),
               "r"(acc));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}\n"
                 : "=r"(done)
                 : "r"(mbar), "r"(parity)
                 : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

// ------------------------------------------------------------ layout check
template <int N>
__global__ void __launch_bounds__(128) k_layout(const unsigned char* A, const unsigned char* B, uint32_t* D, int ksteps) {
  // A: [ksteps][128][32], B: [ksteps][N][32] (row-major bytes)
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) unsigned long long mbar;
  constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  const int tid = threadIdx.x, warp = tid >> 5;
  // B canonical K-major: core matrix (8 rows x 16 B) contiguous 128 B;
  // K-adjacent core matrices LBO = 128 apart, 8-row groups SBO = 256 apart
  for (int i = tid; i < ksteps * N * 32; i += 128) {
    const int s = i / (N * 32), r = (i / 32) % N, k = i % 32;
    sm[s * N * 32 + (r / 8) * 256 + (k / 16) * 128 + (r % 8) * 16 + (k % 16)] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(smem_u32(&mbar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  // A stage s at columns 256 + 8 s
  for (int s = 0; s < ksteps; s++) {
    uint32_t v[8];
    for (int c = 0; c < 8; c++) v[c] = reinterpret_cast<const uint32_t*>(A + ((size_t)s * 128 + tid) * 32)[c];
    tmem_st8(tm + ((uint32_t)(32 * warp) << 16) + 256u + 8u * s, v);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    for (int s = 0; s < ksteps; s++)
      mma_ts(tm, tm + 256u + 8u * s, sdesc(smem_u32(sm) + s * N * 32, 128, 256), IDESC, s ? 1u : 0u);
    mma_commit(smem_u32(&mbar));
  }
  mbar_wait(smem_u32(&mbar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c++) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tm + ((uint32_t)(32 * warp) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    D[tid * N + c] = v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int N>
int check_layout() {
  const int ks = 3;
  std::vector<unsigned char> A(ks * 128 * 32), B(ks * N * 32);
  for (auto& x : A) x = rand();
  for (auto& x : B) x = rand();
  unsigned char *dA, *dB;
  uint32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_layout<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, ks * N * 32 + 1024);
  k_layout<N><<<1, 128, ks * N * 32 + 1024>>>(dA, dB, dD, ks);
  std::vector<uint32_t> D(128 * N);
  cudaError_t e = cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("layout N=%d: error %s\n", N, cudaGetErrorString(e));
    return -1;
  }
  int bad = 0;
  for (int m = 0; m < 128; m++)
    for (int n = 0; n < N; n++) {
      uint32_t r = 0;
      for (int s = 0; s < ks; s++)
        for (int k = 0; k < 32; k++) r += (uint32_t)A[(s * 128 + m) * 32 + k] * B[(s * N + n) * 32 + k];
      if (r != D[m * N + n]) {
        if (bad < 4) printf("  mismatch m=%d n=%d want %u got %u\n", m, n, r, D[m * N + n]);
        bad++;
      }
    }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad;
}

// ------------------------------------------------------------ throughput
// MODE 0: MMAs only (A stages written once).  MODE 1: warps 0-3 rewrite the
// stage each MMA consumed (ring of NS stages, full/empty mbarriers); the MMAs
// are issued by warp 4.
template <int N, int MODE>
__global__ void __launch_bounds__(160) k_ts(int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) unsigned long long bar_full[16], bar_empty[16], bar_done;
  constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  constexpr int NS = 16;  // A stages in TMEM (8 columns each), columns 256..383
  constexpr int KS = 8;   // B K-steps resident in smem
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < KS * N * 32 / 4; i += 160) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < NS; i++) {
      mbar_init(smem_u32(&bar_full[i]), 4);
      mbar_init(smem_u32(&bar_empty[i]), 1);
    }
    mbar_init(smem_u32(&bar_done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const int total = iters * 32;
  if (warp < 4) {
    uint32_t v[8];
    for (int c = 0; c < 8; c++) v[c] = (tid * 8 + c) * 2246822519u;
    const uint32_t tq = tm + ((uint32_t)(32 * warp) << 16) + 256u;
    if (MODE != 1) {
      for (int s = 0; s < NS; s++) tmem_st8(tq + 8u * s, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (lane == 0)
        for (int s = 0; s < NS; s++) mbar_arrive(smem_u32(&bar_full[s]));
    } else {
      for (int k = 0; k < total; k++) {
        const int st = k % NS;
        if (k >= NS) mbar_wait(smem_u32(&bar_empty[st]), (uint32_t)((k / NS - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int c = 0; c < 8; c++) v[c] = __byte_perm(v[c], v[(c + 1) & 7], 0x4321 + (k & 1));
        tmem_st8(tq + 8u * st, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_full[st]));
      }
    }
  } else if (lane == 0) {
    for (int k = 0; k < total; k++) {
      const int st = k % NS;
      if (MODE == 1 || k < NS) mbar_wait(smem_u32(&bar_full[st]), (uint32_t)((k / NS) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (MODE == 2)  // four independent accumulators
        mma_ts(tm + (uint32_t)((k & 3) * N), tm + 256u + 8u * st, sdesc(smem_u32(sm) + (k % KS) * N * 32, 128, 256), IDESC, k > 3 ? 1u : 0u);
      else if (MODE == 3)  // one A stage reused by every MMA
        mma_ts(tm, tm + 256u, sdesc(smem_u32(sm) + (k % KS) * N * 32, 128, 256), IDESC, k ? 1u : 0u);
      else
      mma_ts(tm, tm + 256u + 8u * st, sdesc(smem_u32(sm) + (k % KS) * N * 32, 128, 256), IDESC, k ? 1u : 0u);
      if (MODE == 1) mma_commit(smem_u32(&bar_empty[st]));
    }
    mma_commit(smem_u32(&bar_done));
  }
  mbar_wait(smem_u32(&bar_done), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u) sink[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  }
}

template <int N, int MODE>
double run(int iters) {
  const size_t smem = 8 * N * 32 + 1024;
  cudaFuncSetAttribute(k_ts<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms;  // 512 TMEM columns: one CTA per SM
  k_ts<N, MODE><<<grid, 160, smem>>>(2, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_ts<N, MODE><<<grid, 160, smem>>>(iters, sink);
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
  printf("{\"layout_mismatches\": {\"N16\": %d, \"N48\": %d, \"N256\": %d},\n", check_layout<16>(), check_layout<48>(),
         check_layout<256>());
  const int iters = 2000;
  printf(" \"unit\": \"int8 MAC/s\", \"M\": 128, \"K_per_mma\": 32, \"a_operand\": \"tmem\", \"results\": [\n");
#define R(N)                                                                                         \
  printf("  {\"N\": %d, \"mma_only\": %.4e, \"with_tmem_producers\": %.4e, \"cycles_per_mma_at_1965MHz\": [%.1f, %.1f]},\n", N, \
         run<N, 0>(iters), run<N, 1>(iters), 128.0 * N * 32 * 148 * 1.965e9 / run<N, 0>(iters),                \
         128.0 * N * 32 * 148 * 1.965e9 / run<N, 1>(iters));
  R(16) R(32) R(48) R(64) R(96) R(128) R(256)
#define R2(N) printf("  {\"N\": %d, \"four_accumulators\": %.4e, \"same_a_stage\": %.4e},\n", N, run<N, 2>(iters), run<N, 3>(iters));
  R2(16) R2(32) R2(64)
  printf("  {}\n]}\n");
  return 0;
}
