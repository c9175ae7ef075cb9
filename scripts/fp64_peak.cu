// FP64 peak microbenchmarks on the B200 (the codon roofline needs them;
// MEASURED_PEAKS.json only carries HBM and bf16):
//   dfma_kernel: independent DFMA chains (FP64 vector pipe)
//   dmma_kernel: mma.sync.aligned.m8n8k4.row.col.f64 (legacy fp64 tensor path;
//                tcgen05.mma has no f64 kind on sm_100a)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, double a0) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = a0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int k = 0; k < 2; ++k) {
    const int blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
      else dmma_kernel<<<blocks, threads>>>(out, 1e-3);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = k == 0 ? 2.0 * 16 * ITERS * double(blocks) * threads
                            : 2.0 * 8 * 8 * 4 * 8 * double(ITERS) * double(blocks) * (threads / 32);
      if (rep == 2)
        std::printf("{\"kernel\": \"%s\", \"tflops\": %.2f, \"ms\": %.3f, \"sms\": %d}\n", k == 0 ? "dfma" : "dmma_m8n8k4",
                    flops / (ms * 1e-3) / 1e12, ms, sms);
    }
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) std::printf("error: %s\n", cudaGetErrorString(err));
  return 0;
}
