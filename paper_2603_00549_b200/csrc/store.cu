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
#include <algorithm>

#include "common.cuh"

namespace pm2l {
namespace {

using namespace dev;

constexpr int kEncThreads = 256;
constexpr int kEncRows = 4;                       // points per thread
constexpr int kEncTile = kEncThreads * kEncRows;  // points per CTA

__device__ __forceinline__ uint64_t bswap64(uint64_t v) { return bswap64_ext(v); }

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

// ----------------------------------------------------------- batched lookup
// CacheStore.lookup (pm2lat/nascache.py:408-424) for many points at once:
// each query is a binary search over the sorted big-endian record keys, or,
// for a dense store (every point of its grid present), a direct index from
// per-axis searches (then one record read, key re-checked).  A missing point
// gives NaN and the smallest missing query index in *first_missing.
namespace pm2l {
namespace {

struct LookupAxes {
  const uint64_t* ax[4];
  int64_t len[4];
  int dense;
};

__device__ __forceinline__ int cmp_key(const uint64_t* rec, const uint64_t q[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint64_t v = dev::bswap64_ext(rec[j]);
    if (v != q[j]) return v < q[j] ? -1 : 1;
  }
  return 0;
}

__global__ void store_lookup_kernel(const uint64_t* __restrict__ rec, int64_t n_rec, LookupAxes la,
                                    const uint64_t* __restrict__ qs, int64_t nq,
                                    double* __restrict__ out,
                                    unsigned long long* __restrict__ first_missing) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nq;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t q[4] = {qs[4 * i], qs[4 * i + 1], qs[4 * i + 2], qs[4 * i + 3]};
    int64_t hit = -1;
    if (la.dense) {
      int64_t flat = 0;
      bool ok = true;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        int64_t lo = 0, hi = la.len[a];
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (la.ax[a][mid] < q[a]) lo = mid + 1; else hi = mid;
        }
        ok = ok && lo < la.len[a] && la.ax[a][lo] == q[a];
        flat = flat * la.len[a] + lo;
      }
      if (ok && flat < n_rec && cmp_key(rec + 5 * flat, q) == 0) hit = flat;
    } else {
      int64_t lo = 0, hi = n_rec;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int c = cmp_key(rec + 5 * mid, q);
        if (c == 0) { hit = mid; break; }
        if (c < 0) lo = mid + 1; else hi = mid;
      }
    }
    if (hit >= 0) {
      out[i] = __longlong_as_double(static_cast<long long>(dev::bswap64_ext(rec[5 * hit + 4])));
    } else {
      out[i] = dev::qnan();
      atomicMin(first_missing, (unsigned long long)i);
    }
  }
}

}  // namespace

int launch_store_lookup(const uint8_t* records, int64_t n_rec, const uint64_t* const axes[4],
                        const int64_t lens[4], const uint64_t* queries, int64_t nq, double* out,
                        unsigned long long* first_missing, void* stream) {
  if (nq == 0) return 0;
  LookupAxes la{};
  la.dense = axes != nullptr;
  if (la.dense)
    for (int a = 0; a < 4; ++a) { la.ax[a] = axes[a]; la.len[a] = lens[a]; }
  const int nb = int(std::min<int64_t>((nq + 255) / 256, int64_t(sm_count()) * 16));
  store_lookup_kernel<<<nb, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint64_t*>(records), n_rec, la, queries, nq, out, first_missing);
  return int(cudaGetLastError());
}

}  // namespace pm2l
