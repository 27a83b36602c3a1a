// FP64 SIMT (DFMA) vs FP64 tensor (DMMA m8n8k4) throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[4][2] = {};
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 4; k++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; k++) s += c[k][0] + c[k][1];
  if (s == 12345.0) out[0] = s;
}

// half the warps of each CTA run the DFMA loop, the other half the DMMA
// loop: if the two pipes are separate units the time stays near the time of
// one half alone (SURVEY roofline: is FP64 SIMT + DMMA additive on B200?)
__global__ void mixed_kernel(double *out, int iters_f, int iters_m, int mode) {
  const int w = threadIdx.x >> 5;
  const bool fma_warp = (w & 1) == 0;
  double s = 0;
  if (fma_warp && (mode & 1)) {
    double a[8], b = 1.0000001, c = 0.9999999;
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_f; it++) {
#pragma unroll
      for (int i = 0; i < 8; i++) a[i] = fma(a[i], b, c);
    }
    for (int i = 0; i < 8; i++) s += a[i];
  } else if (!fma_warp && (mode & 2)) {
    double a = threadIdx.x * 1e-3, b = 1.0001;
    double c[4][2] = {};
    for (int it = 0; it < iters_m; it++) {
#pragma unroll
      for (int k = 0; k < 4; k++)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    for (int k = 0; k < 4; k++) s += c[k][0] + c[k][1];
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  double *d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; rep++) {
    int blocks = sms * 8, threads = 256;
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    // m8n8k4: 2*8*8*4 = 512 flops per warp-instruction
    flops = 512.0 * 4 * iters * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  {
    // per warp: DFMA loop = 8*iters_f warp-DFMAs (256 flop each... 2*32*8*iters_f),
    // DMMA loop = 4*iters_m mma (512 flop each)
    const int itf = 20000, itm = 20000 / 4;  // equal flops per warp
    int blocks = sms * 8, threads = 256;
    float t[4] = {0, 0, 0, 0};
    for (int mode = 1; mode <= 3; mode++) {
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        mixed_kernel<<<blocks, threads>>>(d, itf, itm, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t[mode], e0, e1);
      }
      double fl = 0;
      if (mode & 1) fl += 2.0 * 32 * 8 * itf * (double)blocks * (threads / 64);
      if (mode & 2) fl += 512.0 * 4 * itm * (double)blocks * (threads / 64);
      printf("mixed mode %d (1 DFMA half, 2 DMMA half, 3 both): %.3f ms, %.2f TFLOP/s\n", mode, t[mode], fl / t[mode] / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
