// Explicit-descriptor mode: n ops given as 16-byte {b, m, n, k} records.
//   points_kernel        ConfigResolver.resolve (pm2lat/compute.py:251-268):
//                        exact record first, else the nearest record by
//                        Chebyshev distance in log2 space (first scan index
//                        on ties), then the canonical prediction
//                        (compute.py:163-193)
//   points_curve_kernel  predict_generic with an explicit curve (no resolution)
//
// Per op the nearest search uses the same decomposition as the grid kernel —
// member classes and the outward k-group sweep — but without a shared row,
// so D_j(m, n) is recomputed per op from the class members staged in shared
// memory (broadcast reads: all lanes read the same member).
#include <algorithm>

#include "common.cuh"

namespace pm2l {
namespace {

using namespace dev;

__device__ int exact_lookup(const TablesDev& t, uint64_t b, uint64_t m, uint64_t n, uint64_t k,
                            int* curve, int* record) {
  int lo = 0, hi = t.n_exact;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint64_t* e = t.ex_coord + 4 * mid;
    const bool eq = e[0] == b && e[1] == m && e[2] == n && e[3] == k;
    if (eq) {
      *curve = t.ex_curve[mid];
      *record = t.ex_rec[mid];
      return 1;
    }
    const bool less = e[0] != b ? e[0] < b : e[1] != m ? e[1] < m : e[2] != n ? e[2] < n : e[3] < k;
    if (less) lo = mid + 1; else hi = mid;
  }
  return 0;
}

struct PointSmem {
  const double* lm;
  const double* ln;
  const double* glk;
  const int32_t* gcls;
  const int32_t* gstart;
  const int32_t* cstart;
  const int32_t* csize;
  const int32_t* gidx;
};

__device__ __forceinline__ uint64_t member_d(const PointSmem& S, int j, double qm, double qn) {
  return umax64(abs_bits(__dsub_rn(S.lm[j], qm)), abs_bits(__dsub_rn(S.ln[j], qn)));
}

__device__ __forceinline__ uint64_t class_min(const PointSmem& S, int c, double qm, double qn) {
  uint64_t dmin = ~0ull;
  const int s = S.cstart[c], e = s + S.csize[c];
  for (int j = s; j < e; ++j) {
    const uint64_t d = member_d(S, j, qm, qn);
    dmin = d < dmin ? d : dmin;
  }
  return dmin;
}

// first member (scan order) of group g whose D <= best -> candidate scan index
__device__ __forceinline__ int first_within(const PointSmem& S, int g, uint64_t best, double qm,
                                            double qn) {
  const int c = S.gcls[g], s = S.cstart[c], e = s + S.csize[c];
  for (int j = s; j < e; ++j)
    if (member_d(S, j, qm, qn) <= best) return S.gidx[S.gstart[g] + (j - s)];
  return 0x7FFFFFFF;  // unreachable when best >= the class minimum
}

template <bool G32>
__device__ int nearest_point(const TablesDev& t, const PointSmem& S, double qm, double qn,
                             double qk, uint64_t* out_best) {
  // insertion point of qk among the ascending group lk values
  int lo = 0, hi = t.G;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S.glk[mid] < qk) lo = mid + 1; else hi = mid;
  }
  uint64_t best = ~0ull;
  uint32_t mask = 0;
  int best_i = 0x7FFFFFFF;
  int cached = -1;
  uint64_t cached_min = 0;
  auto visit = [&](int g) -> bool {
    const uint64_t dk = abs_bits(__dsub_rn(S.glk[g], qk));
    if (dk > best) return false;
    const int c = S.gcls[g];
    if (c != cached) {
      cached = c;
      cached_min = class_min(S, c, qm, qn);
    }
    const uint64_t dg = umax64(dk, cached_min);
    if (G32) {
      if (dg < best) { best = dg; mask = 1u << g; }
      else if (dg == best) mask |= 1u << g;
    } else if (dg <= best) {
      const int idx = first_within(S, g, dg, qm, qn);
      if (dg < best || idx < best_i) best_i = idx;
      best = dg;
    }
    return true;
  };
  for (int g = lo; g < t.G; ++g)
    if (!visit(g)) break;
  for (int g = lo - 1; g >= 0; --g)
    if (!visit(g)) break;
  if (G32) {
    while (mask) {
      const int g = __ffs(mask) - 1;
      mask &= mask - 1;
      const int idx = first_within(S, g, best, qm, qn);
      best_i = idx < best_i ? idx : best_i;
    }
  }
  *out_best = best;
  return best_i;
}

// One member class (every shipped preset; equal logs imply equal
// coordinates): the grid kernel's nearest_one_class decision per op, with
// the row part from ONE pass over the members -- dmin and its first member
// (case A: mn(k) <= dmin) and the first member within mn(k) (case B).
// Returns the original candidate scan index; *out_best = the distance.
__device__ int nearest_point_one_class(const TablesDev& t, const PointSmem& S, double qm,
                                       double qn, double qk, uint64_t* out_best) {
  const int G = t.G;
  int lo = 0, hi = G;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S.glk[mid] < qk) lo = mid + 1; else hi = mid;
  }
  const int start = lo;
  auto dk = [&](int g) { return abs_bits(__dsub_rn(S.glk[g], qk)); };
  const uint64_t dkL = start > 0 ? dk(start - 1) : ~0ull;
  const uint64_t dkR = start < G ? dk(start) : ~0ull;
  const uint64_t mn = dkL < dkR ? dkL : dkR;
  const int CM = S.csize[0];
  // distances are non-negative finite doubles, so FP64 order is the order
  // of their |.| bits (member_d): compare them as doubles (DMNMX / DSETP)
  const double mnd = __longlong_as_double(static_cast<long long>(mn));
  double dminf = __longlong_as_double(0x7FF0000000000000ll);  // +inf
  int argmin = 0, first_mn = -1;
  for (int j = 0; j < CM; ++j) {
    const double d = fmax(fabs(__dsub_rn(S.lm[j], qm)), fabs(__dsub_rn(S.ln[j], qn)));
    if (d < dminf) { dminf = d; argmin = j; }
    if (first_mn < 0 && d <= mnd) first_mn = j;
  }
  const uint64_t dmin = abs_bits(dminf);
  int g, pos;
  uint64_t best;
  if (mn <= dmin) {  // best == dmin: the leftmost group within dmin, member argmin
    if (dkL <= dmin) {
      g = start - 1;
      while (g > 0 && dk(g - 1) <= dmin) --g;
    } else {
      g = start;
    }
    pos = argmin;
    best = dmin;
  } else {           // best == mn: the leftmost nearest group, first member within mn
    if (dkL == mn) {
      g = start - 1;
      while (g > 0 && dk(g - 1) == mn) --g;
    } else {
      g = start;
    }
    pos = first_mn;
    best = mn;
  }
  *out_best = best;
  return S.gidx[S.gstart[g] + pos];
}

template <int NEARK>  // 0 general sweep, 1 sweep + tie mask (G <= 32), 2 one member class
__global__ void __launch_bounds__(kThreads) points_kernel(TablesDev t, const uint4* __restrict__ shapes,
                                                          int64_t n, const double* __restrict__ lut,
                                                          int64_t lut_n, double* __restrict__ out_lat,
                                                          int32_t* __restrict__ out_curve,
                                                          uint32_t* __restrict__ out_waves,
                                                          int8_t* __restrict__ out_match,
                                                          int32_t* __restrict__ out_record,
                                                          double* __restrict__ out_dist) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* lm = reinterpret_cast<double*>(smem);
  double* ln = lm + t.CM;
  double* glk = ln + t.CM;
  int32_t* gcls = reinterpret_cast<int32_t*>(glk + t.G);
  int32_t* gstart = gcls + t.G;
  int32_t* cstart = gstart + t.G;
  int32_t* csize = cstart + t.NC;
  int32_t* gidx = csize + t.NC;
  for (int j = threadIdx.x; j < t.CM; j += blockDim.x) {
    lm[j] = t.cls_lm[j];
    ln[j] = t.cls_ln[j];
  }
  for (int j = threadIdx.x; j < t.G; j += blockDim.x) {
    glk[j] = t.grp_lk[j];
    gcls[j] = t.grp_class[j];
    gstart[j] = t.grp_start[j];
  }
  for (int j = threadIdx.x; j < t.NC; j += blockDim.x) {
    cstart[j] = t.cls_start[j];
    csize[j] = t.cls_size[j];
  }
  for (int j = threadIdx.x; j < t.R; j += blockDim.x) gidx[j] = t.g_idx[j];
  __syncthreads();
  const PointSmem S{lm, ln, glk, gcls, gstart, cstart, csize, gidx};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 s = shapes[i];
    const uint64_t b = s.x, m = s.y, nn = s.z, k = s.w;
    int ci = -1, rec = -1;
    int8_t match = -1;
    double dist = 0.0;
    if (s.x == 0 || s.y == 0 || s.z == 0 || s.w == 0 || s.y >= lut_n || s.z >= lut_n ||
        s.w >= lut_n) {
      match = -2;  // invalid coordinate (0, or beyond the libm log2 table)
    } else if (exact_lookup(t, b, m, nn, k, &ci, &rec)) {
      match = 0;
    } else if (t.R > 0) {
      uint64_t best;
      rec = NEARK == 2 ? nearest_point_one_class(t, S, lut[s.y], lut[s.z], lut[s.w], &best)
                       : nearest_point<NEARK == 1>(t, S, lut[s.y], lut[s.z], lut[s.w], &best);
      ci = t.cand_curve[rec];
      dist = __longlong_as_double(static_cast<long long>(best));
      match = 1;
    }
    if (out_record) out_record[i] = rec;
    if (out_dist) out_dist[i] = dist;
    if (out_match) out_match[i] = match;
    if (ci < 0) {
      out_lat[i] = qnan();
      if (out_curve) out_curve[i] = -1;
      if (out_waves) out_waves[i] = 0;
      continue;
    }
    const PointResult r = predict_point(t, ci, b, m, nn, k, base_of(t, ci, k));
    out_lat[i] = r.lat;
    if (out_curve) out_curve[i] = ci;
    if (out_waves) out_waves[i] = uint32_t(r.waves);
  }
}

__global__ void points_curve_kernel(TablesDev t, const uint4* __restrict__ shapes,
                                    const int32_t* __restrict__ curves, int64_t n,
                                    double* __restrict__ out_lat, uint32_t* __restrict__ out_waves,
                                    double* __restrict__ out_detail) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 s = shapes[i];
    const int c = curves[i];
    if (c < 0 || c >= t.C || !curve_valid(t, c)) {
      out_lat[i] = qnan();
      if (out_waves) out_waves[i] = 0;
      continue;
    }
    const double nd = __ull2double_rn(uint64_t(s.w));
    const double thr = interp_thr(t, c, nd);
    const double base = base_from_thr(t, c, nd, thr);
    const PointResult r = predict_point(t, c, s.x, s.y, s.z, s.w, base);
    out_lat[i] = r.lat;
    if (out_waves) out_waves[i] = uint32_t(r.waves);
    if (out_detail) {  // Prediction.components: base_us, new_throughput, wave_scale, blocks
      out_detail[4 * i] = base;
      out_detail[4 * i + 1] = thr;
      out_detail[4 * i + 2] = wave_scale(t, c, r.waves);
      out_detail[4 * i + 3] = __ull2double_rn(r.blocks);
    }
  }
}

}  // namespace

int launch_points(const TablesDev& t, const uint32_t* shapes, int64_t n, const double* lut,
                  int64_t lut_n, double* out_lat, int32_t* out_curve, uint32_t* out_waves,
                  int8_t* out_match, int32_t* out_record, double* out_dist, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t smem = 16ll * t.CM + 8ll * t.G + 8ll * t.G + 8ll * t.NC + 4ll * t.R + 64;
  auto* fn = (t.NC == 1 && t.lowest_wins) ? points_kernel<2>
             : t.G <= 32 ? points_kernel<1> : points_kernel<0>;
  if (smem > 227 * 1024) return int(cudaErrorInvalidValue);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return int(e);
  }
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(sm_count()) * 8));
  fn<<<nb, kThreads, smem, s>>>(t, reinterpret_cast<const uint4*>(shapes), n, lut, lut_n, out_lat,
                                out_curve, out_waves, out_match, out_record, out_dist);
  return int(cudaGetLastError());
}

int launch_points_curve(const TablesDev& t, const uint32_t* shapes, const int32_t* curves, int64_t n,
                        double* out_lat, uint32_t* out_waves, double* out_detail, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(sm_count()) * 16));
  points_curve_kernel<<<nb, kThreads, 0, s>>>(t, reinterpret_cast<const uint4*>(shapes), curves, n,
                                             out_lat, out_waves, out_detail);
  return int(cudaGetLastError());
}

}  // namespace pm2l
