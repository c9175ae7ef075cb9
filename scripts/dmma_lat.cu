// DMMA (mma.sync m8n8k4 f64) dependent-chain latency and throughput vs the
// number of independent accumulator chains per warp and warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_lat dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, long long* cyc, int iters) {
  double d[C][2];
#pragma unroll
  for (int c = 0; c < C; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-9 + c;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 0.999;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int warps_per_sm, double* out, long long* dcyc, int sms) {
  const int iters = 4096;
  int threads = 32 * warps_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chains<C><<<sms, threads>>>(out, dcyc, iters);
  cudaEventRecord(e0);
  chains<C><<<sms, threads>>>(out, dcyc, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc;
  cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  double flops = 512.0 * C * iters * double(sms) * warps_per_sm;
  std::printf("{\"chains\": %d, \"warps_per_sm\": %d, \"cycles_per_dmma_per_warp\": %.2f, \"tflops\": %.2f}\n", C,
              warps_per_sm, double(cyc) / (double(iters) * C), flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* dcyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&dcyc, 8);
  for (int w : {1, 4, 8, 16}) {
    run<1>(w, out, dcyc, sms);
    run<2>(w, out, dcyc, sms);
    run<3>(w, out, dcyc, sms);
    run<4>(w, out, dcyc, sms);
    run<6>(w, out, dcyc, sms);
    run<8>(w, out, dcyc, sms);
  }
  return 0;
}
