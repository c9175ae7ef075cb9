// Shared-memory wavefronts per warp-wide load for the access shapes of the
// 4-state walk (uniform P-block loads, 4-address tip-column gathers) at 8-
// and 16-byte widths.  Run under ncu with
//   --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum
// one launch per shape; each launch does ITER loads per warp.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITER = 1024;
template <int W, int MODE>
__global__ void k(double* out) {
  __shared__ __align__(16) double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned h = (lane * 2654435761u) >> 7;
  int off;  // byte offset
  if (MODE == 0) off = 0;                          // uniform
  else if (MODE == 1) off = (lane & 3) * 32;       // 4 addresses, lane % 4
  else if (MODE == 2) off = (h & 3) * 32;          // 4 addresses, scattered over lanes
  else off = lane * W;                             // coalesced
  double acc = 0;
  const char* base = reinterpret_cast<const char*>(sm);
  for (int it = 0; it < ITER; ++it) {
    const int o = off + ((it & 7) * 256);
    if (W == 16) {
      double2 v;
      asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(unsigned(__cvta_generic_to_shared(base + o))));
      acc += v.x + v.y;
    } else {
      double v;
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(unsigned(__cvta_generic_to_shared(base + o))));
      acc += v;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 128 * sizeof(double));
  k<16, 0><<<148, 128>>>(out);
  k<16, 1><<<148, 128>>>(out);
  k<16, 2><<<148, 128>>>(out);
  k<16, 3><<<148, 128>>>(out);
  k<8, 0><<<148, 128>>>(out);
  k<8, 1><<<148, 128>>>(out);
  k<8, 2><<<148, 128>>>(out);
  k<8, 3><<<148, 128>>>(out);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
}
