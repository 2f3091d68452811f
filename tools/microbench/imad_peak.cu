// IMAD.WIDE.U32 throughput microbenchmark (the roofline denominator for the
// multiprecision multiply kernels).  Each thread runs ACC independent 96-bit
// column accumulators fed by 32x32->64 products, exactly the instruction mix
// of the schoolbook multiply (IMAD.WIDE.U32 with carry-out + IADD3.X that
// absorbs two carries).  Also times a plain 64-bit IMAD.WIDE accumulate and a
// plain 32-bit IMAD for reference.  Prints one JSON line.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ACC 8
#define INNER 64

__device__ __forceinline__ void mac96(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t a, uint32_t b) {
  asm volatile("mad.lo.cc.u32 %0,%3,%4,%0;\n\tmadc.hi.cc.u32 %1,%3,%4,%1;\n\taddc.u32 %2,%2,0;"
               : "+r"(c0), "+r"(c1), "+r"(c2) : "r"(a), "r"(b));
}

__global__ void k_mac96(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t c0[ACC], c1[ACC], c2[ACC], bv[ACC];
  uint32_t a = in[threadIdx.x & 31];
#pragma unroll
  for (int r = 0; r < ACC; r++) { c0[r] = c1[r] = c2[r] = 0; bv[r] = in[(threadIdx.x + r) & 63]; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < INNER / ACC; j++) {
#pragma unroll
      for (int r = 0; r < ACC; r++) mac96(c0[r], c1[r], c2[r], a, bv[r]);
      a = a * 0x9E3779B9u + 1u;   // keep operands live (1 IMAD per ACC products)
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int r = 0; r < ACC; r++) s ^= c0[r] ^ c1[r] ^ c2[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_wide64(const uint32_t* in, uint32_t* out, int iters) {
  uint64_t acc[ACC]; uint32_t bv[ACC];
  uint32_t a = in[threadIdx.x & 31];
#pragma unroll
  for (int r = 0; r < ACC; r++) { acc[r] = 0; bv[r] = in[(threadIdx.x + r) & 63]; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < INNER / ACC; j++) {
#pragma unroll
      for (int r = 0; r < ACC; r++) acc[r] += (uint64_t)a * bv[r];
      a = a * 0x9E3779B9u + 1u;
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int r = 0; r < ACC; r++) s ^= acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(s ^ (s >> 32));
}

__global__ void k_imad32(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t acc[ACC], bv[ACC];
  uint32_t a = in[threadIdx.x & 31];
#pragma unroll
  for (int r = 0; r < ACC; r++) { acc[r] = 0; bv[r] = in[(threadIdx.x + r) & 63]; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < INNER / ACC; j++) {
#pragma unroll
      for (int r = 0; r < ACC; r++) acc[r] += a * bv[r];
      a = a * 0x9E3779B9u + 1u;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int r = 0; r < ACC; r++) s ^= acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef void (*kfn)(const uint32_t*, uint32_t*, int);

static double run(kfn k, int blocks, int threads, int iters, const uint32_t* in, uint32_t* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) k<<<blocks, threads>>>(in, out, iters);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(in, out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double products = (double)blocks * threads * iters * INNER;
  return products / (best * 1e-3);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  uint32_t *in, *out; cudaMalloc(&in, 256 * 4); cudaMalloc(&out, (size_t)sms * 64 * 1024 * 4);
  uint32_t h[256]; for (int i = 0; i < 256; i++) h[i] = 0x12345678u * (i + 1) ^ 0xdeadbeefu;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  int iters = 4096;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d, \"results\": [", p.name, sms, clk_khz);
  const char* names[3] = {"mac96_imadwide_cc", "imadwide_u64_acc", "imad_u32"};
  kfn ks[3] = {k_mac96, k_wide64, k_imad32};
  bool first = true;
  for (int ki = 0; ki < 3; ki++) {
    for (int tpb : {256, 512, 1024}) {
      for (int bps : {1, 2, 4}) {
        if (tpb * bps > 2048) continue;
        double r = run(ks[ki], sms * bps, tpb, iters, in, out);
        cudaError_t err = cudaGetLastError();
        printf("%s{\"kernel\": \"%s\", \"tpb\": %d, \"blocks_per_sm\": %d, \"products_per_s\": %.4e, \"err\": \"%s\"}",
               first ? "" : ", ", names[ki], tpb, bps, r, cudaGetErrorString(err));
        first = false;
      }
    }
  }
  printf("]}\n");
  return 0;
}
