// Store encoder: the NAS cache's fixed-width records
// (pm2lat/nascache.py:308-333; format pkg/README.md:117-126) built on the
// device -- four big-endian u64 coordinates (batch, m, n, k) and a
// big-endian f64 latency per RESOLVED point, in canonical grid order
// (unresolved NaN points are dropped, the skip_unresolved semantics).
//
//   store_count_kernel   non-NaN count of each 1024-point tile
//   store_scan_kernel    exclusive scan of the tile counts (one CTA)
//   store_encode_kernel  per tile: ballot/warp-prefix compaction, byte-swap,
//                        five 8-byte stores per record
#include "common.cuh"

namespace pm2l {
namespace {

using namespace dev;

constexpr int kEncThreads = 256;
constexpr int kEncRows = 4;                       // points per thread
constexpr int kEncTile = kEncThreads * kEncRows;  // points per CTA

__device__ __forceinline__ uint64_t bswap64(uint64_t v) {
  const uint32_t lo = uint32_t(v), hi = uint32_t(v >> 32);
  return (uint64_t(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
}

struct EncAxes {
  const uint64_t *B, *M, *N, *K;
  int64_t nM, nN, nK;
};

__global__ void __launch_bounds__(kEncThreads) store_count_kernel(const double* __restrict__ lat,
                                                                  int64_t n, int32_t* counts) {
  __shared__ int32_t warp_sum[kEncThreads / 32];
  const int64_t t0 = int64_t(blockIdx.x) * kEncTile;
  int c = 0;
#pragma unroll
  for (int j = 0; j < kEncRows; ++j) {
    const int64_t p = t0 + j * kEncThreads + threadIdx.x;
    c += (p < n && lat[p] == lat[p]) ? 1 : 0;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kEncThreads / 32; ++w) s += warp_sum[w];
    counts[blockIdx.x] = s;
  }
}

// exclusive scan of `nt` tile counts into offs[0..nt], offs[nt] = total
__global__ void __launch_bounds__(1024) store_scan_kernel(const int32_t* __restrict__ counts,
                                                          int64_t nt, int64_t* __restrict__ offs) {
  __shared__ int64_t part[1024];
  const int64_t per = (nt + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = min(nt, lo + per);
  int64_t s = 0;
  for (int64_t i = lo; i < hi; ++i) s += counts[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < int(blockDim.x); ++i) {
      const int64_t v = part[i];
      part[i] = run;
      run += v;
    }
    offs[nt] = run;
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int64_t i = lo; i < hi; ++i) {
    offs[i] = run;
    run += counts[i];
  }
}

__global__ void __launch_bounds__(kEncThreads) store_encode_kernel(const double* __restrict__ lat,
                                                                   int64_t n, EncAxes ax,
                                                                   const int64_t* __restrict__ offs,
                                                                   uint64_t* __restrict__ rec) {
  __shared__ int32_t warp_base[kEncThreads / 32];
  __shared__ int32_t row_base;
  const int64_t t0 = int64_t(blockIdx.x) * kEncTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = offs[blockIdx.x];
  if (threadIdx.x == 0) row_base = 0;
  for (int j = 0; j < kEncRows; ++j) {
    const int64_t p = t0 + j * kEncThreads + threadIdx.x;
    const double v = p < n ? lat[p] : qnan();
    const bool keep = v == v;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, keep);
    if (lane == 0) warp_base[warp] = __popc(m);
    __syncthreads();
    int wb = 0, tot = 0;
    for (int w = 0; w < kEncThreads / 32; ++w) {
      const int c = warp_base[w];
      wb += w < warp ? c : 0;
      tot += c;
    }
    const int64_t r = base + row_base + wb + __popc(m & ((1u << lane) - 1u));
    if (keep) {
      int64_t q = p;
      const int64_t ik = q % ax.nK; q /= ax.nK;
      const int64_t jn = q % ax.nN; q /= ax.nN;
      const int64_t im = q % ax.nM; q /= ax.nM;
      uint64_t* o = rec + 5 * r;
      o[0] = bswap64(ax.B[q]);
      o[1] = bswap64(ax.M[im]);
      o[2] = bswap64(ax.N[jn]);
      o[3] = bswap64(ax.K[ik]);
      o[4] = bswap64(uint64_t(__double_as_longlong(v)));
    }
    __syncthreads();  // warp_base / row_base reuse
    if (threadIdx.x == 0) row_base += tot;
    __syncthreads();
  }
}

}  // namespace

int64_t store_encode_workspace(int64_t n) {
  const int64_t nt = (n + kEncTile - 1) / kEncTile;
  return nt * 4 + (nt + 1) * 8 + 16;  // counts (i32), offsets (i64)
}

int launch_store_encode(const double* lat, int64_t n, const uint64_t* B, const uint64_t* M,
                        int64_t nM, const uint64_t* N, int64_t nN, const uint64_t* K, int64_t nK,
                        void* workspace, uint8_t* records, int64_t* count, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return int(cudaMemsetAsync(count, 0, sizeof(int64_t), s));
  const int64_t nt = (n + kEncTile - 1) / kEncTile;
  if (nt > 0x7FFFFFFFll) return int(cudaErrorInvalidValue);
  EncAxes ax{B, M, N, K, nM, nN, nK};
  uint64_t* rec = reinterpret_cast<uint64_t*>(records);
  int32_t* counts = static_cast<int32_t*>(workspace);
  int64_t* offs = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(counts + nt) + 15) & ~uintptr_t(15));
  store_count_kernel<<<unsigned(nt), kEncThreads, 0, s>>>(lat, n, counts);
  store_scan_kernel<<<1, 1024, 0, s>>>(counts, nt, offs);
  store_encode_kernel<<<unsigned(nt), kEncThreads, 0, s>>>(lat, n, ax, offs, rec);
  cudaError_t e = cudaMemcpyAsync(count, offs + nt, sizeof(int64_t), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return int(e);
  return int(cudaGetLastError());
}

}  // namespace pm2l
