// the two off-path scans, on the device:
//   grid_error_kernel      curvefit.grid_error_report (pm2lat/curvefit.py:192-219):
//                          per sample interval, the worst relative error of
//                          the piecewise-linear interpolation against a truth
//                          curve over the (strided) integer scan
//   partition_cut_kernel   partition.partition_two_device (pm2lat/partition.py:
//                          53-100): stage sums of every cut, each evaluated
//                          left to right (_ltr_sum) as the reference does,
//   partition_best_kernel  and the first cut of minimum bottleneck.
#include <cstdint>

#include "common.cuh"

namespace pm2l {
namespace {

using namespace dev;

struct ErrKey {
  double err;
  int64_t dim;
};

// the reference's sequential "if err > local[0]" over an ascending scan keeps
// the FIRST maximum: larger error wins, equal errors go to the smaller dim,
// NaN never wins (NaN > x is false)
__device__ __forceinline__ bool better(const ErrKey& a, const ErrKey& b) {
  return a.err > b.err || (a.err == b.err && a.dim < b.dim);
}

// One CTA per sample interval [lo, hi): scan = range(lo, hi, stride), plus hi
// when the range does not end on it (curvefit.py:205-208).  truth: the host
// values of the caller's oracle in scan order (interval i starting at
// scan_off[i]) or, when null, the rational (a*x + b) / (c*x + d) evaluated
// in FP64 left to right as PlantedCurve.__call__ / RationalFit.__call__ do.
constexpr int kMaxAuditSamples = 1024;

__global__ void grid_error_kernel(const int64_t* __restrict__ dims,
                                  const double* __restrict__ thrs, int ns, int64_t stride,
                                  const double* __restrict__ truth,
                                  const int64_t* __restrict__ scan_off, double ra, double rb,
                                  double rc, double rd, double* __restrict__ out_err,
                                  int64_t* __restrict__ out_arg) {
  __shared__ double dimsf[kMaxAuditSamples], thr_s[kMaxAuditSamples];
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    dimsf[i] = __ll2double_rn(dims[i]);
    thr_s[i] = thrs[i];
  }
  __syncthreads();
  const int iv = blockIdx.x;
  const int64_t lo = dims[iv], hi = dims[iv + 1];
  const int64_t n_range = (hi - lo + stride - 1) / stride;
  const bool tail = lo + (n_range - 1) * stride != hi;
  const int64_t count = n_range + (tail ? 1 : 0);
  ErrKey best{-1.0, lo};
  for (int64_t j = threadIdx.x; j < count; j += blockDim.x) {
    const int64_t dim = j < n_range ? lo + j * stride : hi;
    const double x = __ll2double_rn(dim);
    const double tr = truth ? truth[scan_off[iv] + j]
                            : __ddiv_rn(__dadd_rn(__dmul_rn(ra, x), rb),
                                        __dadd_rn(__dmul_rn(rc, x), rd));
    const double it = interp_samples(dimsf, thr_s, 0, ns, x);
    const ErrKey k{__ddiv_rn(fabs(__dsub_rn(it, tr)), tr), dim};
    if (better(k, best)) best = k;
  }
  __shared__ double s_err[256];
  __shared__ int64_t s_dim[256];
  s_err[threadIdx.x] = best.err;
  s_dim[threadIdx.x] = best.dim;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const ErrKey o{s_err[threadIdx.x + w], s_dim[threadIdx.x + w]};
      const ErrKey m{s_err[threadIdx.x], s_dim[threadIdx.x]};
      if (better(o, m)) {
        s_err[threadIdx.x] = o.err;
        s_dim[threadIdx.x] = o.dim;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out_err[iv] = s_err[0];
    out_arg[iv] = s_dim[0];
  }
}

// One thread per cut in [0, n]: stage A = layers [0, cut) of device A,
// stage B = layers [cut, n) of device B (+ the per-cut transfer), each a
// left-to-right FP64 sum from 0.0 (partition.py:53-57), and
// bottleneck = max(stage_a, stage_b) with Python's max (the first argument
// unless the second is greater).
__global__ void partition_cut_kernel(const double* __restrict__ la, const double* __restrict__ lb,
                                     int64_t n, const double* __restrict__ transfer,
                                     double* __restrict__ sa, double* __restrict__ sb,
                                     double* __restrict__ bn) {
  const int64_t cut = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (cut > n) return;
  double a = 0.0, b = 0.0;
  for (int64_t i = 0; i < cut; ++i) a = __dadd_rn(a, la[i]);
  for (int64_t i = cut; i < n; ++i) b = __dadd_rn(b, lb[i]);
  b = __dadd_rn(b, transfer ? transfer[cut] : 0.0);
  sa[cut] = a;
  sb[cut] = b;
  bn[cut] = b > a ? b : a;
}

// The reference's scan "if best is None or bottleneck < best" (partition.py:
// 90-94): cut 0 first, replaced only by a strictly smaller bottleneck -- the
// first minimum; NaN never replaces (and a NaN at cut 0 is never replaced).
__global__ void partition_best_kernel(const double* __restrict__ bn, int64_t n,
                                      int64_t* __restrict__ best) {
  __shared__ double s_v[256];
  __shared__ int64_t s_i[256];
  double v = __longlong_as_double(0x7FF0000000000000ll);
  int64_t idx = INT64_MAX;
  for (int64_t c = threadIdx.x; c <= n; c += blockDim.x) {
    const double x = bn[c];
    if (x < v || (x == v && c < idx)) {
      v = x;
      idx = c;
    }
  }
  s_v[threadIdx.x] = v;
  s_i[threadIdx.x] = idx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double ov = s_v[threadIdx.x + w];
      const int64_t oi = s_i[threadIdx.x + w];
      if (ov < s_v[threadIdx.x] || (ov == s_v[threadIdx.x] && oi < s_i[threadIdx.x])) {
        s_v[threadIdx.x] = ov;
        s_i[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double b0 = bn[0];
    // cut 0 wins outright when its bottleneck is NaN (nothing compares
    // below it) or when nothing is strictly below it
    *best = (b0 != b0 || !(s_v[0] < b0)) ? 0 : s_i[0];
  }
}

}  // namespace

int launch_grid_error(const int64_t* dims, const double* thrs, int ns, int64_t stride,
                      const double* truth, const int64_t* scan_off, const double* rational,
                      double* out_err, int64_t* out_arg, void* stream) {
  if (ns < 2) return 0;
  if (ns > kMaxAuditSamples || stride < 1) return int(cudaErrorInvalidValue);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const double r0 = rational ? rational[0] : 0.0, r1 = rational ? rational[1] : 0.0;
  const double r2 = rational ? rational[2] : 0.0, r3 = rational ? rational[3] : 1.0;
  grid_error_kernel<<<ns - 1, 256, 0, s>>>(dims, thrs, ns, stride, truth, scan_off, r0, r1, r2,
                                           r3, out_err, out_arg);
  return int(cudaGetLastError());
}

int launch_partition(const double* la, const double* lb, int64_t n, const double* transfer,
                     double* sa, double* sb, double* bn, int64_t* best, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t cuts = n + 1;
  partition_cut_kernel<<<int((cuts + 127) / 128), 128, 0, s>>>(la, lb, n, transfer, sa, sb, bn);
  partition_best_kernel<<<1, 256, 0, s>>>(bn, n, best);
  return int(cudaGetLastError());
}

}  // namespace pm2l
