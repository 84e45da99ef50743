// Primitive-cost microbenchmarks on B200 (sm_100a): decides how the
// level kernels rank and count keys.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kIters = 4096;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void k_match(uint32_t* out, int nb_mask) {
  uint32_t acc = 0, v = hash32(threadIdx.x + blockIdx.x * 977);
  for (int i = 0; i < kIters; ++i) {
    v = v * 1664525u + 1013904223u;
    acc += __match_any_sync(0xffffffffu, (v >> 8) & nb_mask);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int BITS>
__global__ void k_ballot_match(uint32_t* out, int nb_mask) {
  uint32_t acc = 0, v = hash32(threadIdx.x + blockIdx.x * 977);
  for (int i = 0; i < kIters; ++i) {
    v = v * 1664525u + 1013904223u;
    const uint32_t b = (v >> 8) & nb_mask;
    uint32_t m = 0xffffffffu;
#pragma unroll
    for (int bit = 0; bit < BITS; ++bit) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (b >> bit) & 1);
      m &= ((b >> bit) & 1) ? bal : ~bal;
    }
    acc += m;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_atom_spread(uint32_t* out, int nb_mask) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < (nb_mask + 1) * (int)(blockDim.x / 32); i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t v = hash32(threadIdx.x + blockIdx.x * 977);
  uint32_t* hw = h + (threadIdx.x >> 5) * (nb_mask + 1);
  for (int i = 0; i < kIters; ++i) {
    v = v * 1664525u + 1013904223u;
    atomicAdd(&hw[(v >> 8) & nb_mask], 1u);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x & nb_mask];
}

__global__ void k_atom_same(uint32_t* out, int) {
  __shared__ uint32_t h[32];
  if (threadIdx.x < 32) h[threadIdx.x] = 0;
  __syncthreads();
  uint32_t v = hash32(threadIdx.x + blockIdx.x * 977);
  for (int i = 0; i < kIters; ++i) {
    v = v * 1664525u + 1013904223u;
    atomicAdd(&h[(threadIdx.x >> 5) & 7], v & 1);
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x & 31];
}

// per-lane private u16 counters [bucket][lane] per warp
__global__ void k_lane_counters(uint32_t* out, int nb_mask) {
  extern __shared__ uint16_t c16[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint16_t* cw = c16 + (size_t)w * (nb_mask + 1) * 32;
  for (int i = threadIdx.x; i < (nb_mask + 1) * 32 * (blockDim.x / 32); i += blockDim.x) c16[i] = 0;
  __syncthreads();
  uint32_t v = hash32(threadIdx.x + blockIdx.x * 977);
  for (int i = 0; i < kIters; ++i) {
    v = v * 1664525u + 1013904223u;
    uint16_t* p = cw + ((v >> 8) & nb_mask) * 32 + lane;
    *p = *p + 1;
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = c16[threadIdx.x & nb_mask];
}

__global__ void k_alu(uint32_t* out, int nb_mask) {
  uint32_t acc = 0, v = hash32(threadIdx.x + blockIdx.x * 977);
  for (int i = 0; i < kIters; ++i) {
    v = v * 1664525u + 1013904223u;
    acc += (v >> 8) & nb_mask;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_read(const uint4* __restrict__ in, size_t n16, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = in[i];
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void k_copy(const uint4* __restrict__ in, uint4* __restrict__ o, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    o[i] = in[i];
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  uint32_t* out;
  CK(cudaMalloc(&out, 64 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int threads = 256, blocks = sms * 8;
  auto run = [&](const char* name, auto fn, int nb_mask, size_t smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<blocks, threads, smem>>>(out, nb_mask);
    cudaEventRecord(a);
    fn<<<blocks, threads, smem>>>(out, nb_mask);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * kIters;  // lane-ops
    double cyc_per_warpop = (ms * 1e-3) * clk * 1e3 * sms / (ops / 32);
    printf("%-28s nb=%5d  %.3f ms  %.2f Glane-op/s  %.2f SM-cycles per warp-op\n", name, nb_mask + 1,
           ms, ops / ms / 1e6, cyc_per_warpop);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  err %s\n", cudaGetErrorString(e));
  };
  run("alu baseline", k_alu, 127, 0);
  run("match_any.b32", k_match, 127, 0);
  run("match_any.b32", k_match, 4095, 0);
  run("ballot-match 7 bits", k_ballot_match<7>, 127, 0);
  run("ballot-match 9 bits", k_ballot_match<9>, 511, 0);
  run("atomicAdd smem per-warp", k_atom_spread, 127, 8 * 128 * 4);
  run("atomicAdd smem per-warp", k_atom_spread, 1023, 8 * 1024 * 4);
  run("atomicAdd smem same addr", k_atom_same, 0, 0);
  run("lane u16 counters", k_lane_counters, 127, 8 * 128 * 32 * 2);
  run("lane u16 counters", k_lane_counters, 255, 8 * 256 * 32 * 2);
  // memory
  size_t bytes = (size_t)4 << 30;
  uint4* buf; uint4* buf2;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&buf2, bytes));
  cudaMemset(buf, 1, bytes);
  size_t n16 = bytes / 16;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_read<<<sms * 16, 512>>>(buf, n16, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("stream read  %.1f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(a);
    k_copy<<<sms * 16, 512>>>(buf, buf2, n16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("copy (r+w)   %.1f GB/s\n", 2 * bytes / ms / 1e6);
  }
  printf("sms=%d clock=%d kHz\n", sms, clk);
  return 0;
}
