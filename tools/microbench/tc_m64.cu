// tc_swz.cu with M = 64 MMAs: where do the 64 rows land in TMEM, and what does an M = 64 step cost?
// Byte convolution on tcgen05.mma kind::i8 with NO per-K-step operand build:
//
//   A = sliding windows over the raw bytes of a, stored once with the
//       hardware swizzle (SWIZZLE_32B / 64B / 128B => row pitch 32 / 64 / 128
//       bytes, so M = 128 rows span 128 * pitch byte positions),
//   B = N = pitch shifted, reversed copies of b, read through ONE table of
//       8 byte phases T[x][r][i] = b[r + c - 8x - i] with LBO = 256, SBO = 128
//       (row n = r + 8g of K-step s is entry x = 4s + g + 2q: linear in g and q).
//
// Checks D = conv(a, b) on a tile against the host, for two base_offset
// conventions of the descriptor, then times the MMA stream.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_swz tc_swz.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// K-major descriptor: layout type lt (0 none, 2 128B, 4 64B, 6 32B), base offset bo
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t lt, uint32_t bo) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)(bo & 7u) << 49) | ((uint64_t)lt << 61);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc),
               "r"(acc));
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  long long spins = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}\n"
                 : "=r"(done)
                 : "r"(mbar), "r"(parity)
                 : "memory");
    if (++spins > 20000000ll) { printf("mbar timeout\n"); __trap(); }
  } while (!done);
}
__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

__host__ __device__ inline int fdiv32(int x) { return x >= 0 ? x / 32 : -((-x + 31) / 32); }

template <int PITCH>
struct G {
  static constexpr int N = PITCH;
  static constexpr int LT = PITCH == 128 ? 2 : PITCH == 64 ? 4 : 6;
  static constexpr int MASK = PITCH / 16 - 1;  // swizzle: bits [4, 4+B) ^= bits [7, 7+B)
  static constexpr int AMAX = 127 * PITCH;
  static constexpr int PADL = AMAX + 64;
  static constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (4u << 24);  // M = 64
};

// MODE 0: correctness (D written out), MODE 1: timing (reps products per CTA)
template <int PITCH, int MODE>
__global__ void __launch_bounds__(128) k_conv(const unsigned char* a, const unsigned char* b, int La, int Lb, int tile,
                                              int bo_mode, uint32_t* D, int reps, unsigned long long* sink) {
  using g = G<PITCH>;
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) unsigned long long mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  // 1024-aligned base
  unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  const int T = 128 * PITCH;
  const int ntiles = (La + Lb - 1 + T - 1) / T;
  const int ulo = -32 * ((Lb - 1 + 31) / 32);
  const int S = fdiv32(g::N - 1 - ulo) + 1;
  const int PADR = ntiles * T + 64 - La > 64 ? ntiles * T + 64 - La : 64;
  const int asz = (g::PADL + La + PADR + 1023) & ~1023;
  unsigned char* abuf = sm;            // logical byte x of [pad | a | pad] at swizzled address
  unsigned char* tab = sm + asz;       // T[x]: 128 bytes per entry
  const int X = 4 * S + g::N / 8 + 2;
  const uint32_t abase = smem_u32(abuf);
  for (int x = tid; x < asz; x += 128) {
    const int j = x - g::PADL;
    const unsigned char v = (j >= 0 && j < La) ? a[j] : 0;
    const uint32_t L = abase + x;
    const uint32_t P = L ^ (((L >> 7) & g::MASK) << 4);
    abuf[P - abase] = v;
  }
  const int cc = g::N - 8 - ulo;
  for (int e = tid; e < X * 128; e += 128) {
    const int x = e >> 7, r = (e >> 4) & 7, i = e & 15;
    const int j = r + cc - 8 * x - i;
    tab[e] = (j >= 0 && j < Lb) ? b[j] : 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(128));
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
  const int k0 = tile * T;
  int slo = -fdiv32(k0 + g::AMAX + 31 + ulo);
  if (slo < 0) slo = 0;
  int shi = fdiv32(La - k0 - 1 - ulo) + 1;
  if (shi > S) shi = S;
  if (tid == 0) {
    uint32_t phase = 0;
    for (int rep = 0; rep < reps; rep++) {
      for (int s = slo; s < shi; s++) {
        const uint32_t start = abase + (uint32_t)(g::PADL + k0 + ulo + 32 * s);
        const uint32_t bo = bo_mode ? (start >> 7) & 7u : 0u;
        const uint64_t ad = sdesc(start, 16, 8 * PITCH, g::LT, bo);
        const uint64_t bd = sdesc(smem_u32(tab) + 512u * (uint32_t)s, 256, 128, 0, 0);
        mma_i8(tm, ad, bd, g::IDESC, s > slo ? 1u : 0u);
      }
      mma_commit(smem_u32(&mbar));
      mbar_wait(smem_u32(&mbar), phase);
      phase ^= 1;
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (MODE == 0) {
    for (int c = 0; c < g::N; c++) {
      uint32_t v;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n"
                   : "=r"(v)
                   : "r"(tm + ((uint32_t)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      D[tid * g::N + c] = v;
    }
  } else if (warp == 0) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u && tid == 0) sink[0] = v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}

template <int PITCH>
size_t smem_need(int La, int Lb) {
  using g = G<PITCH>;
  const int T = 128 * PITCH;
  const int ntiles = (La + Lb - 1 + T - 1) / T;
  const int ulo = -32 * ((Lb - 1 + 31) / 32);
  const int S = fdiv32(g::N - 1 - ulo) + 1;
  const int PADR = ntiles * T + 64 - La > 64 ? ntiles * T + 64 - La : 64;
  const int asz = (g::PADL + La + PADR + 1023) & ~1023;
  return (size_t)asz + (size_t)(4 * S + g::N / 8 + 2) * 128 + 1024;
}

template <int PITCH>
int check(int La, int Lb, int tile, int bo_mode) {
  using g = G<PITCH>;
  std::vector<unsigned char> a(La), b(Lb);
  for (auto& x : a) x = rand();
  for (auto& x : b) x = rand();
  unsigned char *da, *db;
  uint32_t* dD;
  unsigned long long* sink;
  cudaMalloc(&da, La);
  cudaMalloc(&db, Lb);
  cudaMalloc(&dD, 128 * g::N * 4);
  cudaMalloc(&sink, 8);
  cudaMemcpy(da, a.data(), La, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), Lb, cudaMemcpyHostToDevice);
  const size_t smem = smem_need<PITCH>(La, Lb);
  cudaFuncSetAttribute(k_conv<PITCH, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_conv<PITCH, 0><<<1, 128, smem>>>(da, db, La, Lb, tile, bo_mode, dD, 1, sink);
  std::vector<uint32_t> D(128 * g::N);
  cudaError_t e = cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("  error %s\n", cudaGetErrorString(e));
    return -1;
  }
  int bad = 0;
  // expected rows of an M = 64 tile; find which TMEM lane holds each
  std::vector<std::vector<uint32_t>> want(64, std::vector<uint32_t>(g::N));
  for (int m = 0; m < 64; m++)
    for (int n = 0; n < g::N; n++) {
      const int beta = (n % 8) - 8 * (n / 8) + g::N - 8;
      const int k = tile * 128 * PITCH + PITCH * m + beta;
      uint32_t r = 0;
      for (int j = 0; j < Lb; j++) {
        const int i = k - j;
        if (i >= 0 && i < La) r += (uint32_t)a[i] * b[j];
      }
      want[m][n] = r;
    }
  printf("  lane->row:");
  for (int L = 0; L < 128; L++) {
    int found = -1;
    for (int m = 0; m < 64; m++) {
      bool eq = true;
      for (int n = 0; n < g::N; n++) eq &= want[m][n] == D[L * g::N + n];
      if (eq) { found = m; break; }
    }
    if (found < 0) bad++;
    printf(" %d", found);
  }
  printf("\n");
  cudaFree(da);
  cudaFree(db);
  cudaFree(dD);
  cudaFree(sink);
  return bad;
}

template <int PITCH>
void timeit(int La, int Lb, int ctas_per_sm) {
  using g = G<PITCH>;
  unsigned char *da, *db;
  unsigned long long* sink;
  cudaMalloc(&da, La);
  cudaMalloc(&db, Lb);
  cudaMalloc(&sink, 8);
  cudaMemset(da, 0x5a, La);
  cudaMemset(db, 0xa5, Lb);
  const size_t smem = smem_need<PITCH>(La, Lb);
  cudaFuncSetAttribute(k_conv<PITCH, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 200;
  k_conv<PITCH, 1><<<sms * ctas_per_sm, 128, smem>>>(da, db, La, Lb, 0, 0, nullptr, 2, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_conv<PITCH, 1><<<sms * ctas_per_sm, 128, smem>>>(da, db, La, Lb, 0, 0, nullptr, reps, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t e = cudaGetLastError();
  const int ulo = -32 * ((Lb - 1 + 31) / 32);
  const int S = fdiv32(g::N - 1 - ulo) + 1;
  int slo = -fdiv32(g::AMAX + 31 + ulo);
  if (slo < 0) slo = 0;
  int shi = fdiv32(La - 1 - ulo) + 1;
  if (shi > S) shi = S;
  const double mmas = (double)(shi - slo) * reps * sms * ctas_per_sm;
  const double cyc = ms * 1e-3 * 1.965e9 * sms / mmas;  // SM-cycles per MMA
  printf("  {\"pitch_N\": %d, \"La\": %d, \"Lb\": %d, \"ctas_per_sm\": %d, \"smem\": %zu, \"mmas_per_product\": %d, "
         "\"sm_cycles_per_mma\": %.1f, \"us_per_product_per_sm\": %.3f, \"issued_mac_per_s\": %.4e, \"err\": \"%s\"},\n",
         PITCH, La, Lb, ctas_per_sm, smem, shi - slo, cyc, ms * 1e3 * sms / (reps * sms * ctas_per_sm),
         mmas * 64.0 * g::N * 32 / (ms * 1e-3), e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(da);
  cudaFree(db);
  cudaFree(sink);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int idx = 0;
  printf("{\"layout_mismatches\": [\n");
#define C(P, La, Lb, t)                                                                                          \
  if (only < 0 || only == idx++) printf("  {\"pitch\": %d, \"La\": %d, \"Lb\": %d, \"tile\": %d, \"base_offset_0\": %d, \"base_offset_addr\": %d},\n", P, La, \
         Lb, t, check<P>(La, Lb, t, 0), check<P>(La, Lb, t, 1));
  C(64, 2436, 2436, 0)
  printf("  {}],\n \"timing\": [\n");
  if (only >= 0 && only < 100) return 0;
  int t = 100;
#define TM(P, La, Lb, C) if (only < 0 || only == t++) timeit<P>(La, Lb, C);
  TM(64, 2436, 2436, 1) TM(64, 2436, 2436, 2) TM(64, 2436, 2436, 3) TM(32, 2436, 2436, 3) TM(128, 2436, 2436, 2)
  printf("  {}]}\n");
  return 0;
}
