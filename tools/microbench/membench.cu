// Microbenchmarks used to size the chebfd kernel design on B200 (sm_100a):
// HBM stream, L2-resident and L1-resident 512-B row gathers, FP64 FMA rate.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void copy_cs(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) __stcs(b + i, __ldcs(a + i));
}
__global__ void read_sum(const double2* __restrict__ a, size_t n, double* out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  double s = 0;
  for (; i < n; i += st) { double2 v = __ldcs(a + i); s += v.x + v.y; }
  if (s == 1234.5) *out = s;
}
// Each warp: rows of 32 x double2 = 512 B. 13 gathers per "row step" from a buffer of nrows rows.
template <int MODE>
__global__ void gather13(const double2* __restrict__ u, unsigned nrows, unsigned mask_region, int iters, double* out) {
  int lane = threadIdx.x & 31;
  unsigned w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned base = (MODE == 2) ? (blockIdx.x * 97u) % nrows : 0;  // L1 mode: per-CTA small region
  unsigned h = w * 2654435761u + 12345u;
  double2 acc = make_double2(0, 0);
  for (int it = 0; it < iters; ++it) {
    double2 v[13];
#pragma unroll
    for (int k = 0; k < 13; ++k) {
      h = h * 1664525u + 1013904223u;
      unsigned r = (MODE == 2) ? (base + ((h >> 8) & mask_region)) % nrows : (h >> 4) % nrows;
      const double2* p = u + (size_t)r * 32 + lane;
      if (MODE == 1) v[k] = __ldcg(p); else v[k] = __ldg(p);
    }
#pragma unroll
    for (int k = 0; k < 13; ++k) { acc.x += v[k].x; acc.y += v[k].y; }
  }
  if (acc.x == 1234.5) *out = acc.y;
}
__global__ void dfma_rate(double* out, int iters) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5) *out = s;
}
int main() {
  int dev = 0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, dev));
  printf("device %s SMs %d L2 %d MB smemPerSM %zu KB clock %d MHz memclk %d MHz bus %d\n", pr.name, pr.multiProcessorCount,
         pr.l2CacheSize >> 20, pr.sharedMemPerMultiprocessor >> 10, pr.clockRate / 1000, pr.memoryClockRate / 1000, pr.memoryBusWidth);
  size_t n = (size_t)1 << 28;  // 256M double2 = 4 GiB
  double2 *a, *b; double* out;
  CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16)); CK(cudaMalloc(&out, 8));
  CK(cudaMemset(a, 0, n * 16)); CK(cudaMemset(b, 0, n * 16));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = pr.multiProcessorCount;
  float ms;
  for (int bpsm : {2, 4, 8}) {
    for (int r = 0; r < 2; ++r) copy_cs<<<sms * bpsm, 512>>>(a, b, n);
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) copy_cs<<<sms * bpsm, 512>>>(a, b, n); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("copy_cs bpsm=%d: %.1f GB/s\n", bpsm, 5.0 * 2 * n * 16 / (ms * 1e-3) / 1e9);
  }
  for (int r = 0; r < 2; ++r) read_sum<<<sms * 8, 512>>>(a, n, out);
  cudaEventRecord(e0); for (int r = 0; r < 5; ++r) read_sum<<<sms * 8, 512>>>(a, n, out); cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
  printf("read_sum: %.1f GB/s\n", 5.0 * n * 16 / (ms * 1e-3) / 1e9);
  int iters = 64;
  for (int mb : {8, 32, 64, 96, 128, 256, 4096}) {
    unsigned nrows = (unsigned)(((size_t)mb << 20) / 512);
    for (int mode = 0; mode < 2; ++mode) {
      for (int warps : {16, 32, 48}) {
        int blocks = sms * warps / 8;
        auto launch = [&]() { if (mode == 0) gather13<0><<<blocks, 256>>>(a, nrows, 0, iters, out); else gather13<1><<<blocks, 256>>>(a, nrows, 0, iters, out); };
        launch(); launch();
        cudaEventRecord(e0); for (int r = 0; r < 3; ++r) launch(); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double bytes = 3.0 * blocks * 8.0 * iters * 13 * 512;
        printf("gather13 %s buf=%4d MB warps/SM=%d: %.1f GB/s delivered\n", mode ? "cg(L2)" : "nc(L1)", mb, warps, bytes / (ms * 1e-3) / 1e9);
      }
    }
  }
  for (int reg : {63, 255, 1023, 4095}) {  // per-CTA region rows (512 B each): 32KB .. 2MB
    unsigned nrows = (unsigned)((256u << 20) / 512);
    int blocks = sms * 2;
    auto launch = [&]() { gather13<2><<<blocks, 512>>>(a, nrows, reg, iters, out); };
    launch();
    cudaEventRecord(e0); for (int r = 0; r < 3; ++r) launch(); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 3.0 * blocks * 16.0 * iters * 13 * 512;
    printf("gather13 L1-region %d KB per CTA (2 CTA/SM, 32 warps/SM): %.1f GB/s delivered\n", (reg + 1) / 2, bytes / (ms * 1e-3) / 1e9);
  }
  {
    int it2 = 4096;
    dfma_rate<<<sms * 8, 256>>>(out, it2);
    cudaEventRecord(e0); dfma_rate<<<sms * 8, 256>>>(out, it2); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("dfma: %.2f TFLOP/s (fp64, 2 flop/fma)\n", 2.0 * sms * 8 * 256.0 * it2 * 8 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
