// Site-pattern compression on the GPU: the
// first-occurrence compression of SitePatternAlignment::from_codes
// (/root/reference/proj/include/phylograd/alignment.hpp:186-229) for
// alignments that are too large to compress quickly on the host (C3: 2048 taxa
// x 10^6 columns).  Integer work, bit-exact with the host path:
//
//   K_hash16  one thread per 16 columns: validate codes (-1..m-1) and hash
//             the columns top to bottom, 16-byte loads of 4 taxa per step
//             transposed in registers into 4-taxon column words;
//   K_insert  open-addressing table keyed by the 64-bit hash; the slot keeps
//             the smallest column index (atomicMin) = the first occurrence;
//   K_verify  every column is compared byte for byte with its representative,
//             so a hash collision can never merge different columns (a
//             collision re-runs the whole pass with another seed);
//   scan      representatives get pattern ids in increasing column order,
//             which IS the reference's first-occurrence order;
//   K_finish  site -> pattern map and integer weights (atomic counts: exact);
//   K_gather  pattern codes [ntax][P] gathered from the representative
//             columns.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <memory>
#include <string>

#include "pg_common.hpp"

namespace {

using pg::CudaError;
using pg::NotSupported;

#define PGC_CUDA(call)                                                                                 \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess) throw CudaError(std::string("cuda: ") + #call + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
struct DBuf {
  T* p = nullptr;
  explicit DBuf(size_t n) { PGC_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

constexpr unsigned long long kEmpty = ~0ull;
constexpr int kScanBlock = 1024;

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// One thread per group of 16 consecutive columns (rows padded to a multiple
// of 16 bytes): each step loads one 16-byte chunk from each of 4 taxa
// (512 contiguous bytes per warp per taxon), validates the 64 codes with SIMD
// byte compares, transposes them into 16 column words of 4 taxa (8 PRMT per 4
// columns) and mixes each word into its column's 64-bit hash.
__device__ __forceinline__ void mix_word(uint64_t& x, uint32_t w) {
  x = (x ^ w) * 0x9E3779B97F4A7C15ull;
  x ^= x >> 29;
}

__global__ void k_hash16(const int8_t* __restrict__ codes, int ntax, int S, int pitch, int m, uint64_t seed,
                         unsigned long long* __restrict__ h, int* bad) {
  const int groups = (S + 15) / 16;
  const uint32_t mm = uint32_t(m) * 0x01010101u;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < groups; j += gridDim.x * blockDim.x) {
    uint64_t x[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) x[c] = seed;
    uint32_t badm = 0;
    const int ncols = min(16, S - 16 * j);
#pragma unroll 2
    for (int t = 0; t < ntax; t += 4) {
      uint4 v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        v[r] = t + r < ntax ? __ldcs(reinterpret_cast<const uint4*>(codes + size_t(t + r) * pitch) + j)
                            : make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      const uint32_t* a = reinterpret_cast<const uint32_t*>(v);  // a[r * 4 + q]: taxon t+r, columns 4q..4q+3
#pragma unroll
      for (int i = 0; i < 16; ++i) badm |= __vcmpgtu4(__vadd4(a[i], 0x01010101u), mm);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t t0 = __byte_perm(a[q], a[4 + q], 0x5140), t1 = __byte_perm(a[q], a[4 + q], 0x7362);
        const uint32_t t2 = __byte_perm(a[8 + q], a[12 + q], 0x5140), t3 = __byte_perm(a[8 + q], a[12 + q], 0x7362);
        mix_word(x[4 * q + 0], __byte_perm(t0, t2, 0x5410));
        mix_word(x[4 * q + 1], __byte_perm(t0, t2, 0x7632));
        mix_word(x[4 * q + 2], __byte_perm(t1, t3, 0x5410));
        mix_word(x[4 * q + 3], __byte_perm(t1, t3, 0x7632));
      }
    }
    if (badm) {
      // locate the first bad column of this group (rare path)
      for (int c = 0; c < ncols; ++c)
        for (int t = 0; t < ntax; ++t) {
          const int v = codes[size_t(t) * pitch + 16 * j + c];
          if (v < -1 || v >= m) {
            atomicMin(bad, 16 * j + c);
            t = ntax;
            c = ncols;
          }
        }
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const unsigned long long v = fmix64(x[c] ^ uint64_t(ntax));
      if (c < ncols) h[16 * j + c] = v == kEmpty ? kEmpty - 1 : v;
    }
  }
}

__global__ void k_insert(const unsigned long long* __restrict__ h, int S, unsigned long long* keys, int* vals,
                         unsigned long long mask, unsigned* __restrict__ slot_of) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const unsigned long long k = h[s];
    unsigned long long slot = k & mask;
    for (;;) {
      const unsigned long long cur = atomicCAS(keys + slot, kEmpty, k);
      if (cur == kEmpty || cur == k) break;
      slot = (slot + 1) & mask;
    }
    atomicMin(vals + slot, s);
    slot_of[s] = unsigned(slot);
  }
}

__global__ void k_verify(const int8_t* __restrict__ codes, int ntax, int S, int pitch, const int* __restrict__ vals,
                         const unsigned* __restrict__ slot_of, int* __restrict__ rep, int* __restrict__ flag,
                         int* collisions) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const int r = vals[slot_of[s]];
    rep[s] = r;
    flag[s] = r == s;
    if (r != s) {
      for (int t = 0; t < ntax; ++t)
        if (codes[size_t(t) * pitch + s] != codes[size_t(t) * pitch + r]) {
          atomicAdd(collisions, 1);
          break;
        }
    }
  }
}

// exclusive scan of flag[] in blocks of kScanBlock; block totals to bsum[]
__global__ void k_scan_blocks(const int* __restrict__ flag, int S, int* __restrict__ out, int* __restrict__ bsum) {
  __shared__ int warp_tot[32];
  const int i = blockIdx.x * kScanBlock + threadIdx.x;
  const int v = i < S ? flag[i] : 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const int before = (w > 0 ? warp_tot[w - 1] : 0) + x - v;
  if (i < S) out[i] = before;
  if (threadIdx.x == kScanBlock - 1) bsum[blockIdx.x] = warp_tot[31];
}

// one block: exclusive scan of the block totals (any count, chunked), total to *total
__global__ void k_scan_bsum(int* bsum, int nb, int* total) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < nb; base += kScanBlock) {
    const int i = base + threadIdx.x;
    const int v = i < nb ? bsum[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      int t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
    }
    __syncthreads();
    const int c = carry;
    if (i < nb) bsum[i] = c + (w > 0 ? warp_tot[w - 1] : 0) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry = c + warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_finish(int S, const int* __restrict__ rep, const int* __restrict__ local,
                         const int* __restrict__ bsum, int* __restrict__ site_to_pattern,
                         unsigned long long* __restrict__ weights, int* __restrict__ rep_site) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const int r = rep[s];
    const int pid = local[r] + bsum[r / kScanBlock];
    site_to_pattern[s] = pid;
    atomicAdd(weights + pid, 1ull);
    if (r == s) rep_site[pid] = s;
  }
}

// 16 patterns per thread: 16 bytes of one taxon, one 16-byte store (output
// rows padded to a multiple of 16 bytes).  When the 16 representative
// columns are consecutive (the common case: mostly unique columns) the bytes
// come from two aligned 16-byte loads and a funnel shift; otherwise they are
// gathered one by one.
__global__ void k_gather(const int8_t* __restrict__ codes, int ntax, int pitch, int P, int opitch,
                         const int* __restrict__ rep_site, int8_t* __restrict__ out) {
  const int groups = (P + 15) / 16;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += gridDim.x * blockDim.x) {
    const int first = __ldg(rep_site + 16 * g);
    const bool full = 16 * g + 15 < P;
    const bool run = full && __ldg(rep_site + 16 * g + 15) == first + 15;
    const int base = first & ~15, o = first & 15;
    for (int t = blockIdx.y; t < ntax; t += gridDim.y) {
      const int8_t* row = codes + size_t(t) * pitch;
      uint32_t w[4] = {0, 0, 0, 0};
      if (run) {
        const uint4 lo = __ldg(reinterpret_cast<const uint4*>(row + base));
        const uint4 hi = o ? __ldg(reinterpret_cast<const uint4*>(row + base + 16)) : make_uint4(0, 0, 0, 0);
        const uint32_t v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        const int q = o >> 2, sh = 8 * (o & 3);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t a = v[i], b = v[i + 1];
#pragma unroll
          for (int k = 1; k < 4; ++k)
            if (q == k) {
              a = v[i + k];
              b = v[i + k + 1];
            }
          w[i] = __funnelshift_r(a, b, sh);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int p = 16 * g + k;
          const uint32_t b = p < P ? uint8_t(row[__ldg(rep_site + p)]) : 0u;
          w[k >> 2] |= b << (8 * (k & 3));
        }
      }
      reinterpret_cast<uint4*>(out + size_t(t) * opitch)[g] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

struct GpuCompressHandle {
  int device = 0, ntax = 0, S = 0, P = 0, opitch = 16;
  std::unique_ptr<DBuf<int8_t>> pattern_codes;
  std::unique_ptr<DBuf<unsigned long long>> weights;
  std::unique_ptr<DBuf<int>> site_to_pattern;
  float ms = 0.f;
};

}  // namespace

extern "C" {

int pg_compress_codes_gpu(int ntax, int64_t sites, const int8_t* codes, int codes_on_device, int state_count,
                          int device, void** handle, int* pattern_count) {
  return pg::guarded([&] {
    if (state_count < 2) throw std::invalid_argument("alignment: state count must be >= 2");
    if (ntax <= 0) throw std::invalid_argument("alignment: no records");
    if (sites < 0) throw std::invalid_argument("alignment: negative site count");
    if (sites >= 0x7f000000) throw NotSupported("alignment: GPU compression supports < 2^31 - 2^24 columns");
    if (state_count > 126) throw NotSupported("alignment: int8 codes hold at most 126 states");
    PGC_CUDA(cudaSetDevice(device));
    auto H = std::make_unique<GpuCompressHandle>();
    H->device = device;
    H->ntax = ntax;
    H->S = int(sites);
    const int S = H->S;
    cudaStream_t st;
    PGC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    cudaEvent_t e0, e1;
    PGC_CUDA(cudaEventCreate(&e0));
    PGC_CUDA(cudaEventCreate(&e1));
    struct EventGuard {
      cudaEvent_t a, b;
      ~EventGuard() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
    } eg{e0, e1};
    if (S == 0) {
      H->pattern_codes = std::make_unique<DBuf<int8_t>>(0);
      H->weights = std::make_unique<DBuf<unsigned long long>>(0);
      H->site_to_pattern = std::make_unique<DBuf<int>>(0);
      *pattern_count = 0;
      *handle = H.release();
      return;
    }
    // rows padded to 16 bytes (vector loads); the padding is zeroed
    const int pitch = (S + 15) / 16 * 16;
    DBuf<int8_t> pad{size_t(ntax) * size_t(pitch) + 16};
    // outputs sized for the worst case P = S, allocated before the timed region
    const int opitch = pitch;
    H->opitch = opitch;
    H->weights = std::make_unique<DBuf<unsigned long long>>(size_t(S));
    H->site_to_pattern = std::make_unique<DBuf<int>>(size_t(S));
    H->pattern_codes = std::make_unique<DBuf<int8_t>>(size_t(ntax) * size_t(opitch));
    DBuf<int> rep_site{size_t(S)};
    int sms = 0;
    PGC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int T = 256;
    const int G = std::max(1, std::min((S + T - 1) / T, sms * 8));
    unsigned long long cap = 1;
    while (cap < 2ull * unsigned(S)) cap <<= 1;
    DBuf<unsigned long long> h{size_t(S)}, keys{size_t(cap)};
    DBuf<int> vals{size_t(cap)}, rep{size_t(S)}, flag{size_t(S)}, local{size_t(S)}, scal{size_t(4)};
    DBuf<unsigned> slot_of{size_t(S)};
    const int nb = (S + kScanBlock - 1) / kScanBlock;
    DBuf<int> bsum{size_t(nb)};
    if (codes_on_device) PGC_CUDA(cudaEventRecord(e0, st));
    PGC_CUDA(cudaMemcpy2DAsync(pad.p, pitch, codes, size_t(S), size_t(S), size_t(ntax),
                               codes_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    if (pitch > S) PGC_CUDA(cudaMemset2DAsync(pad.p + S, pitch, 0, size_t(pitch - S), size_t(ntax), st));
    if (!codes_on_device) {
      PGC_CUDA(cudaStreamSynchronize(st));  // the pageable H2D copy is not part of the device time
      PGC_CUDA(cudaEventRecord(e0, st));
    }
    const int8_t* dc = pad.p;
    int hs[3];
    for (int attempt = 0;; ++attempt) {
      if (attempt == 4) throw std::runtime_error("alignment: GPU compression: repeated 64-bit hash collisions");
      const int init[3] = {INT_MAX, 0, 0};  // first bad column, collisions, total patterns
      PGC_CUDA(cudaMemcpyAsync(scal.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
      PGC_CUDA(cudaMemsetAsync(keys.p, 0xff, cap * sizeof(unsigned long long), st));
      PGC_CUDA(cudaMemsetAsync(vals.p, 0x7f, cap * sizeof(int), st));  // 0x7f7f7f7f > any column index
      const uint64_t seed = 0x51ed270b27a1f3c5ull + 0x9E3779B97F4A7C15ull * uint64_t(attempt);
      const int groups = (S + 15) / 16;
      k_hash16<<<std::max(1, std::min((groups + 127) / 128, sms * 16)), 128, 0, st>>>(dc, ntax, S, pitch, state_count,
                                                                                     seed, h.p, scal.p);
      k_insert<<<G, T, 0, st>>>(h.p, S, keys.p, vals.p, cap - 1, slot_of.p);
      k_verify<<<G, T, 0, st>>>(dc, ntax, S, pitch, vals.p, slot_of.p, rep.p, flag.p, scal.p + 1);
      PGC_CUDA(cudaGetLastError());
      PGC_CUDA(cudaMemcpyAsync(hs, scal.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
      PGC_CUDA(cudaStreamSynchronize(st));
      if (hs[0] != INT_MAX) throw std::invalid_argument("alignment: state code out of range");
      if (hs[1] == 0) break;
    }
    k_scan_blocks<<<nb, kScanBlock, 0, st>>>(flag.p, S, local.p, bsum.p);
    k_scan_bsum<<<1, kScanBlock, 0, st>>>(bsum.p, nb, scal.p + 2);
    PGC_CUDA(cudaGetLastError());
    PGC_CUDA(cudaMemcpyAsync(hs + 2, scal.p + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
    PGC_CUDA(cudaStreamSynchronize(st));
    const int P = hs[2];
    H->P = P;
    PGC_CUDA(cudaMemsetAsync(H->weights->p, 0, size_t(P) * sizeof(unsigned long long), st));
    k_finish<<<G, T, 0, st>>>(S, rep.p, local.p, bsum.p, H->site_to_pattern->p, H->weights->p, rep_site.p);
    const int pgroups = (P + 15) / 16;
    dim3 gg(unsigned(std::max(1, std::min((pgroups + T - 1) / T, 64))), unsigned(std::min(ntax, 65535)));
    k_gather<<<gg, T, 0, st>>>(dc, ntax, pitch, P, opitch, rep_site.p, H->pattern_codes->p);
    PGC_CUDA(cudaGetLastError());
    PGC_CUDA(cudaEventRecord(e1, st));
    PGC_CUDA(cudaStreamSynchronize(st));
    PGC_CUDA(cudaEventElapsedTime(&H->ms, e0, e1));
    *pattern_count = P;
    *handle = H.release();
  });
}

int pg_compress_result_gpu(void* handle, int8_t* pattern_codes, int64_t* weights, int32_t* site_to_pattern,
                           float* device_ms) {
  return pg::guarded([&] {
    auto* H = static_cast<GpuCompressHandle*>(handle);
    if (!H) throw std::invalid_argument("alignment: null compression handle");
    PGC_CUDA(cudaSetDevice(H->device));
    if (pattern_codes && H->P)
      PGC_CUDA(cudaMemcpy2D(pattern_codes, size_t(H->P), H->pattern_codes->p, size_t(H->opitch), size_t(H->P),
                            size_t(H->ntax), cudaMemcpyDeviceToHost));
    if (weights && H->P) {
      static_assert(sizeof(unsigned long long) == sizeof(int64_t), "weights are 64-bit counts");
      PGC_CUDA(cudaMemcpy(weights, H->weights->p, size_t(H->P) * sizeof(int64_t), cudaMemcpyDeviceToHost));
    }
    if (site_to_pattern && H->S)
      PGC_CUDA(cudaMemcpy(site_to_pattern, H->site_to_pattern->p, size_t(H->S) * sizeof(int32_t),
                          cudaMemcpyDeviceToHost));
    if (device_ms) *device_ms = H->ms;
  });
}

void pg_compress_free_gpu(void* handle) { delete static_cast<GpuCompressHandle*>(handle); }

}  // extern "C"
