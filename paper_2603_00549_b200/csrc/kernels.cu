// sm_100a kernels of the PM2Lat batched latency-prediction path.
//
//   grid_kernel          canonical (b, m, n, k) grid: nearest-config argmin per
//                        (m, n, k) via per-row k-group staircases in shared memory,
//                        integer tile/wave model, per-(curve, k) base table,
//                        one DMUL + one 8-byte coalesced store per point
//   base_table_kernel    base(c, k) = ref_dur*(k/ref_dim)*(ref_thr/thr(c,k))
//   fixup_kernel         exact-record hits (take priority over nearest)
//   all_curves_kernel    shape x every kernel ("mode X")
//   points_kernel        explicit 16-byte op descriptors (resolve + predict)
//   membound_kernel      5-feature FMA-chain linear model with launch floor
//   segment_fsum_kernel  exact (== math.fsum) per-model totals, one warp per model
//
// Arithmetic order is the reference's canonical order (pm2lat/compute.py:109-138,
// _kernels.pyx:50-73,119-132).  Every FP64 op on the latency path is an explicit
// round-to-nearest intrinsic (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn), which
// nvcc never contracts into DFMA; the library is also built with -fmad=false.
// The membound dot product is the one place that NEEDS fused multiply-adds
// (it mirrors OpenBLAS ddot's FMA chain behind np.dot, membound.py:121).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "pm2l_internal.h"

namespace pm2l {

namespace {

constexpr uint64_t kAbsMask = 0x7FFFFFFFFFFFFFFFull;
constexpr int kThreads = 256;

__device__ __forceinline__ uint64_t abs_bits(double x) {
  return static_cast<uint64_t>(__double_as_longlong(x)) & kAbsMask;
}

// (a + b - 1) / b in u64 exactly as the Cython kernel writes it
// (_kernels.pyx:124,126,127); 32-bit hardware path when both operands fit.
__device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) {
  const uint64_t num = a + b - 1;
  if ((num | b) <= 0xFFFFFFFFull) return uint64_t(uint32_t(num) / uint32_t(b));
  return num / b;
}

// compute._interpolate_detail / _kernels._interp: clamp outside the sampled
// range, exact at samples, linear between neighbours (no FMA).
__device__ double interp_thr(const TablesDev& t, int c, double nd) {
  const int lo = t.s_off[c], hi = t.s_off[c + 1];
  const double* d = t.s_dims;
  const double* y = t.s_thrs;
  if (nd < d[lo]) return y[lo];
  if (nd > d[hi - 1]) return y[hi - 1];
  int left = lo, right = hi;
  while (left < right) {
    const int mid = (left + right) >> 1;
    if (d[mid] < nd) left = mid + 1; else right = mid;
  }
  if (d[left] == nd) return y[left];
  const double k1 = d[left - 1], k3 = d[left], t1 = y[left - 1], t3 = y[left];
  const double tt = __ddiv_rn(__dsub_rn(nd, k1), __dsub_rn(k3, k1));
  return __dadd_rn(t1, __dmul_rn(tt, __dsub_rn(t3, t1)));
}

// compute._rescale (first factor): base depends on (curve, k) only.
__device__ double base_of(const TablesDev& t, int c, uint64_t k) {
  const double nd = __ull2double_rn(k);
  const double thr = interp_thr(t, c, nd);
  return __dmul_rn(__dmul_rn(t.ref_dur[c], __ddiv_rn(nd, t.ref_dim[c])),
                   __ddiv_rn(t.ref_thr[c], thr));
}

// compute.block_count (78-99) in u64 (Cython semantics, _kernels.pyx:123-126).
__device__ __forceinline__ uint64_t blocks_of(const TablesDev& t, int c, uint64_t b, uint64_t m,
                                              uint64_t n, uint64_t k) {
  const uint64_t tm = t.tile_m[c];
  if (t.rowblock[c]) return ceil_div(b * k, tm);
  return b * ceil_div(m, tm) * ceil_div(n, t.tile_n[c]) * t.split_k[c];
}

__device__ __forceinline__ double wave_scale(const TablesDev& t, int c, uint64_t waves) {
  return __ddiv_rn(__ull2double_rn(waves), t.ref_waves[c]);
}

struct PointResult {
  double lat;
  uint64_t blocks, waves;
};

// Full canonical per-point arithmetic for a known curve (used by fix-ups,
// explicit descriptors, and the general per-point path).
__device__ PointResult predict_point(const TablesDev& t, int c, uint64_t b, uint64_t m,
                                     uint64_t n, uint64_t k, double base) {
  PointResult r;
  r.blocks = blocks_of(t, c, b, m, n, k);
  r.waves = ceil_div(r.blocks, t.bpw[c]);
  r.lat = __dmul_rn(base, wave_scale(t, c, r.waves));
  return r;
}

// ---------------------------------------------------------------- base table
__global__ void base_table_kernel(TablesDev t, const uint64_t* __restrict__ K, int64_t nK,
                                  double* __restrict__ base) {
  const int64_t total = int64_t(t.C) * nK;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(e / nK);
    const int64_t ik = e - int64_t(c) * nK;
    base[e] = (t.s_off[c + 1] > t.s_off[c]) ? base_of(t, c, K[ik]) : 0.0;
  }
}

// --------------------------------------------------------------- grid kernel
// Modes: 0 = GEMM curves, wave scale table W[ib][c] per CTA in smem;
//        1 = GEMM curves, tiles-per-(m,n) table, wave scale per point;
//        2 = general (row-block curves present): everything per point.
struct GridLaunch {
  int kpt;          // k values per thread
  int ktiles;       // k tiles per row
  int nbs;          // batch slabs
  int64_t bper;     // batch values per slab
  int mode;
  int64_t smem;
};

struct SmemLayout {
  int64_t off_D, off_sD, off_sI, off_grp, off_T, off_W, total;
};

// Per-row, per-k-group state in shared memory (32 B: one LDS.128 reads lk+dmin).
struct __align__(16) GroupRow {
  double lk;        // log2 k of the group
  uint64_t dmin;    // min over members of D_i(m, n) (as ordered bits)
  int32_t sstart;   // staircase start (== group start in group order)
  int32_t last;     // scan index of the first member attaining dmin
  int32_t len;      // staircase length
  int32_t pad;
};

__host__ __device__ inline SmemLayout smem_layout(int R, int G, int C, int64_t bper, int mode) {
  SmemLayout L;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t at = o;
    o = (o + bytes + 15) & ~int64_t(15);
    return at;
  };
  L.off_D = take(8ll * R);
  L.off_sD = take(8ll * R);
  L.off_sI = take(4ll * R);
  L.off_grp = take(int64_t(sizeof(GroupRow)) * G);
  L.off_T = take(mode <= 1 ? 8ll * C : 0);
  L.off_W = take(mode == 0 ? 8ll * C * bper : 0);
  L.total = o;
  return L;
}

// Nearest-config argmin for one query k given the row's staircases.
//
// dist(i) = max(D_i, dk_g(i)) with dk_g = |lk_g - qk|.  Groups are sorted by
// lk, so dk_g grows monotonically (IEEE subtraction is monotone) when moving
// away from qk's insertion point `start`: sweep right, then left, stopping a
// side as soon as dk_g exceeds the running best (no member of that group or
// any farther group can reach it).  The minimum scan index among all members
// attaining the final best is then read off the staircases of the tying
// groups: the first staircase entry with D <= best (O(1) when best == dmin).
// Returns the ORIGINAL candidate scan index (INT32_MAX when G == 0).
__device__ __forceinline__ int stair_index(const GroupRow& gr, uint64_t best,
                                           const uint64_t* __restrict__ sD,
                                           const int32_t* __restrict__ sI) {
  if (best == gr.dmin) return gr.last;
  int s = gr.sstart;
  while (sD[s] > best) ++s;
  return sI[s];
}

template <bool G32>
__device__ __forceinline__ int nearest_in_row(int G, double qk, int start,
                                              const GroupRow* __restrict__ grp,
                                              const uint64_t* __restrict__ sD,
                                              const int32_t* __restrict__ sI) {
  uint64_t best = ~0ull;
  uint32_t mask = 0;
  int best_i = 0x7FFFFFFF;
  auto visit = [&](int g) -> bool {
    const double2 lkd = *reinterpret_cast<const double2*>(&grp[g]);
    const uint64_t dk = abs_bits(__dsub_rn(lkd.x, qk));
    if (dk > best) return false;
    const uint64_t gm = static_cast<uint64_t>(__double_as_longlong(lkd.y));
    const uint64_t dg = dk > gm ? dk : gm;
    if (G32) {
      if (dg < best) { best = dg; mask = 1u << g; }
      else if (dg == best) mask |= 1u << g;
    } else if (dg <= best) {
      const int idx = stair_index(grp[g], dg, sD, sI);
      if (dg < best || idx < best_i) best_i = idx;
      best = dg;
    }
    return true;
  };
  for (int g = start; g < G; ++g)
    if (!visit(g)) break;
  for (int g = start - 1; g >= 0; --g)
    if (!visit(g)) break;
  if (G32) {
    while (mask) {
      const int g = __ffs(mask) - 1;
      mask &= mask - 1;
      const int idx = stair_index(grp[g], best, sD, sI);
      best_i = idx < best_i ? idx : best_i;
    }
  }
  return best_i;
}

template <bool VERIFY, int MODE, bool G32>
__global__ void __launch_bounds__(kThreads) grid_kernel(TablesDev t, GridDev g, GridLaunch gl,
                                                        const double* __restrict__ base_tab,
                                                        LaunchOut out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const SmemLayout L = smem_layout(t.R, t.G, t.C, gl.bper, MODE);
  uint64_t* sDv = reinterpret_cast<uint64_t*>(smem + L.off_D);
  uint64_t* sD = reinterpret_cast<uint64_t*>(smem + L.off_sD);
  int32_t* sI = reinterpret_cast<int32_t*>(smem + L.off_sI);
  GroupRow* grp = reinterpret_cast<GroupRow*>(smem + L.off_grp);
  uint64_t* Tmn = reinterpret_cast<uint64_t*>(smem + L.off_T);
  double* W = reinterpret_cast<double*>(smem + L.off_W);

  int64_t cta = blockIdx.x;
  const int ks = int(cta % gl.ktiles);
  cta /= gl.ktiles;
  const int bs = int(cta % gl.nbs);
  const int64_t row = cta / gl.nbs;
  const int64_t im = row / g.nN, jn = row - (row / g.nN) * g.nN;
  const int64_t ib0 = g.b_lo + int64_t(bs) * gl.bper;
  const int64_t ib1 = min(g.b_hi, ib0 + gl.bper);
  if (ib0 >= ib1) return;
  const uint64_t m = g.M[im], n = g.N[jn];
  const double qm = g.logM[im], qn = g.logN[jn];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  // 1. D_i = max(|lm_i - qm|, |ln_i - qn|) for every candidate (group order)
  for (int j = tid; j < t.R; j += blockDim.x) {
    const uint64_t a = abs_bits(__dsub_rn(t.g_lm[j], qm));
    const uint64_t b = abs_bits(__dsub_rn(t.g_ln[j], qn));
    sDv[j] = a > b ? a : b;
  }
  for (int j = tid; j < t.G; j += blockDim.x) {
    grp[j].lk = t.grp_lk[j];
    grp[j].sstart = t.grp_start[j];
  }
  if (MODE <= 1) {
    for (int c = tid; c < t.C; c += blockDim.x)
      Tmn[c] = (t.s_off[c + 1] > t.s_off[c])
                   ? ceil_div(m, t.tile_m[c]) * ceil_div(n, t.tile_n[c]) * t.split_k[c]
                   : 0;
  }
  __syncthreads();

  // 2. per group: prefix-minimum staircase of D over the scan order (warp per group)
  for (int gi = warp; gi < t.G; gi += nwarps) {
    const int start = t.grp_start[gi], size = t.grp_size[gi];
    uint64_t carry = ~0ull;
    int len = 0;
    for (int base = 0; base < size; base += 32) {
      const int j = base + lane;
      const uint64_t d = j < size ? sDv[start + j] : ~0ull;
      uint64_t pm = d;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, pm, off);
        if (lane >= off && o < pm) pm = o;
      }
      uint64_t excl = __shfl_up_sync(0xFFFFFFFFu, pm, 1);
      if (lane == 0) excl = ~0ull;
      if (carry < excl) excl = carry;
      const bool rec = (j < size) && (d < excl);
      const unsigned mask = __ballot_sync(0xFFFFFFFFu, rec);
      if (rec) {
        const int pos = start + len + __popc(mask & ((1u << lane) - 1u));
        sD[pos] = d;
        sI[pos] = t.g_idx[start + j];
      }
      len += __popc(mask);
      const uint64_t tail = __shfl_sync(0xFFFFFFFFu, pm, 31);
      if (tail < carry) carry = tail;
    }
    __syncwarp();
    if (lane == 0) {
      grp[gi].dmin = carry;
      grp[gi].len = len;
      grp[gi].last = len ? sI[start + len - 1] : 0x7FFFFFFF;
    }
  }
  // 3. wave-scale table: W[ib][c] = waves(b, m, n, c) / ref_waves[c]
  if (MODE == 0) {
    const int64_t nb = ib1 - ib0;
    for (int64_t e = tid; e < nb * t.C; e += blockDim.x) {
      const int64_t ib = e / t.C;
      const int c = int(e - ib * t.C);
      if (t.s_off[c + 1] > t.s_off[c]) {
        const uint64_t blocks = g.B[ib0 + ib] * Tmn[c];
        W[e] = wave_scale(t, c, ceil_div(blocks, t.bpw[c]));
      }
    }
  }
  __syncthreads();

  // 4. points: each thread owns kpt k values (stride blockDim), all batches
  const int64_t plane = g.nM * g.nN * g.nK;  // elements per batch index
  const int64_t row_off = (im * g.nN + jn) * g.nK;
  const int64_t k0 = int64_t(ks) * gl.kpt * blockDim.x;
  for (int j = 0; j < gl.kpt; ++j) {
    const int64_t ik = k0 + int64_t(j) * blockDim.x + tid;
    if (ik >= g.nK) break;
    const double qk = g.logK[ik];
    const int best = nearest_in_row<G32>(t.G, qk, g.kstart[ik], grp, sD, sI);
    const int ci = (best < t.R) ? t.cand_curve[best] : -1;
    double* o = out.lat + (ib0 - g.b_lo) * plane + row_off + ik;
    if (ci < 0) {
      if (out.nan_stats) {
        atomicMin(out.nan_stats, (unsigned long long)(o - out.lat));
        atomicAdd(out.nan_stats + 1, (unsigned long long)(ib1 - ib0));
      }
      for (int64_t ib = ib0; ib < ib1; ++ib, o += plane) {
        *o = __longlong_as_double(0x7FF8000000000000ll);
        if (VERIFY) {
          const int64_t p = o - out.lat;
          out.curve[p] = -1;
          out.blocks[p] = 0;
          out.waves[p] = 0;
        }
      }
      continue;
    }
    const uint64_t k = g.K[ik];
    const double base = base_tab ? base_tab[int64_t(ci) * g.nK + ik] : base_of(t, ci, k);
    for (int64_t ib = ib0; ib < ib1; ++ib, o += plane) {
      double lat;
      uint64_t blocks = 0, waves = 0;
      if (MODE == 0 && !VERIFY) {
        lat = __dmul_rn(base, W[(ib - ib0) * t.C + ci]);
      } else if (MODE <= 1) {
        blocks = g.B[ib] * Tmn[ci];
        waves = ceil_div(blocks, t.bpw[ci]);
        lat = __dmul_rn(base, wave_scale(t, ci, waves));
      } else {
        const PointResult r = predict_point(t, ci, g.B[ib], m, n, k, base);
        lat = r.lat;
        blocks = r.blocks;
        waves = r.waves;
      }
      *o = lat;
      if (VERIFY) {
        const int64_t p = o - out.lat;
        out.curve[p] = ci;
        out.blocks[p] = blocks;
        out.waves[p] = waves;
      }
    }
  }
}

template <bool VERIFY>
__global__ void fixup_kernel(TablesDev t, GridDev g, LaunchOut out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= g.n_fix) return;
  const int64_t p = g.fix_pos[i];
  const uint64_t* c4 = g.fix_coord + 4 * i;
  const int ci = g.fix_curve[i];
  if (out.nan_stats) {
    // the main kernel counted this point by its nearest result; re-count it
    // by its exact result (fix-ups are rare: <= one per recorded shape).  A
    // NaN that disappears may have been the minimum: flag the stats dirty so
    // the host re-derives the first NaN with nan_scan_kernel.
    const bool was_nan = out.lat[p] != out.lat[p];
    if (was_nan && ci >= 0) {
      atomicAdd(out.nan_stats + 1, ~0ull);  // -1
      atomicOr(out.nan_stats + 2, 1ull);
    }
    if (!was_nan && ci < 0) {
      atomicAdd(out.nan_stats + 1, 1ull);
      atomicMin(out.nan_stats, (unsigned long long)p);
    }
  }
  if (ci < 0) {
    out.lat[p] = __longlong_as_double(0x7FF8000000000000ll);
    if (VERIFY) { out.curve[p] = -1; out.blocks[p] = 0; out.waves[p] = 0; }
    return;
  }
  const PointResult r = predict_point(t, ci, c4[0], c4[1], c4[2], c4[3], base_of(t, ci, c4[3]));
  out.lat[p] = r.lat;
  if (VERIFY) { out.curve[p] = ci; out.blocks[p] = r.blocks; out.waves[p] = r.waves; }
}

// ---------------------------------------------------------- mode X (all curves)
__global__ void __launch_bounds__(kThreads) all_curves_kernel(TablesDev t, GridDev g, GridLaunch gl,
                                                              const double* __restrict__ base_tab,
                                                              double* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* Tmn = reinterpret_cast<uint64_t*>(smem);
  double* W = reinterpret_cast<double*>(smem + ((8ll * t.C + 15) & ~15ll));
  int64_t cta = blockIdx.x;
  const int ks = int(cta % gl.ktiles);
  cta /= gl.ktiles;
  const int bs = int(cta % gl.nbs);
  const int64_t row = cta / gl.nbs;
  const int64_t im = row / g.nN, jn = row - (row / g.nN) * g.nN;
  const int64_t ib0 = g.b_lo + int64_t(bs) * gl.bper;
  const int64_t ib1 = min(g.b_hi, ib0 + gl.bper);
  if (ib0 >= ib1) return;
  const uint64_t m = g.M[im], n = g.N[jn];
  const int tid = threadIdx.x;
  const bool table = gl.mode == 0;
  if (table) {
    for (int c = tid; c < t.C; c += blockDim.x)
      Tmn[c] = (t.s_off[c + 1] > t.s_off[c])
                   ? ceil_div(m, t.tile_m[c]) * ceil_div(n, t.tile_n[c]) * t.split_k[c]
                   : 0;
    __syncthreads();
    for (int64_t e = tid; e < (ib1 - ib0) * t.C; e += blockDim.x) {
      const int64_t ib = e / t.C;
      const int c = int(e - ib * t.C);
      if (t.s_off[c + 1] > t.s_off[c])
        W[e] = wave_scale(t, c, ceil_div(g.B[ib0 + ib] * Tmn[c], t.bpw[c]));
    }
    __syncthreads();
  }
  const int64_t slice = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  const int64_t plane = g.nM * g.nN * g.nK;
  const int64_t row_off = (im * g.nN + jn) * g.nK;
  const int64_t k0 = int64_t(ks) * gl.kpt * blockDim.x;
  for (int j = 0; j < gl.kpt; ++j) {
    const int64_t ik = k0 + int64_t(j) * blockDim.x + tid;
    if (ik >= g.nK) break;
    const uint64_t k = g.K[ik];
    for (int c = 0; c < t.C; ++c) {
      const double base = base_tab[int64_t(c) * g.nK + ik];
      const bool valid = t.s_off[c + 1] > t.s_off[c];
      double* o = out + int64_t(c) * slice + (ib0 - g.b_lo) * plane + row_off + ik;
      for (int64_t ib = ib0; ib < ib1; ++ib, o += plane) {
        double lat;
        if (!valid) lat = __longlong_as_double(0x7FF8000000000000ll);
        else if (table) lat = __dmul_rn(base, W[(ib - ib0) * t.C + c]);
        else lat = predict_point(t, c, g.B[ib], m, n, k, base).lat;
        __stcs(o, lat);
      }
    }
  }
}

// ---------------------------------------------------- explicit descriptors
// Reference ConfigResolver.resolve (compute.py:251-268): exact dict hit first,
// else the first candidate (scan order) minimising the Chebyshev distance.
__device__ int exact_lookup(const TablesDev& t, uint64_t b, uint64_t m, uint64_t n, uint64_t k,
                            int* curve, int* record) {
  int lo = 0, hi = t.n_exact;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint64_t* e = t.ex_coord + 4 * mid;
    bool less = e[0] != b ? e[0] < b : e[1] != m ? e[1] < m : e[2] != n ? e[2] < n : e[3] < k;
    bool eq = e[0] == b && e[1] == m && e[2] == n && e[3] == k;
    if (eq) {
      *curve = t.ex_curve[mid];
      *record = t.ex_rec[mid];
      return 1;
    }
    if (less) lo = mid + 1; else hi = mid;
  }
  return 0;
}

__global__ void __launch_bounds__(kThreads) points_kernel(TablesDev t, const uint4* __restrict__ shapes,
                                                          int64_t n, const double* __restrict__ lut,
                                                          int64_t lut_n,
                                                          double* __restrict__ out_lat,
                                                          int32_t* __restrict__ out_curve,
                                                          uint32_t* __restrict__ out_waves,
                                                          int8_t* __restrict__ out_match,
                                                          int32_t* __restrict__ out_record,
                                                          double* __restrict__ out_dist) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* cLm = reinterpret_cast<double*>(smem);
  double* cLn = cLm + t.R;
  int32_t* cIdx = reinterpret_cast<int32_t*>(cLn + t.R);
  for (int j = threadIdx.x; j < t.R; j += blockDim.x) {
    cLm[j] = t.g_lm[j];
    cLn[j] = t.g_ln[j];
    cIdx[j] = t.g_idx[j];
  }
  __syncthreads();
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
      const double qm = lut[s.y], qn = lut[s.z], qk = lut[s.w];
      uint64_t best_d = ~0ull;
      int best_i = 0x7FFFFFFF;
      for (int gi = 0; gi < t.G; ++gi) {
        const uint64_t dk = abs_bits(__dsub_rn(t.grp_lk[gi], qk));
        if (dk > best_d) continue;  // every member of this group is farther
        const int start = t.grp_start[gi], end = start + t.grp_size[gi];
        for (int j = start; j < end; ++j) {
          const uint64_t a = abs_bits(__dsub_rn(cLm[j], qm));
          const uint64_t bb = abs_bits(__dsub_rn(cLn[j], qn));
          uint64_t d = a > bb ? a : bb;
          d = d > dk ? d : dk;
          const int idx = cIdx[j];
          if (d < best_d || (d == best_d && idx < best_i)) { best_d = d; best_i = idx; }
        }
      }
      ci = t.cand_curve[best_i];
      rec = best_i;
      dist = __longlong_as_double(static_cast<long long>(best_d));
      match = 1;
    }
    if (out_record) out_record[i] = rec;
    if (out_dist) out_dist[i] = dist;
    if (ci < 0) {
      out_lat[i] = __longlong_as_double(0x7FF8000000000000ll);
      if (out_curve) out_curve[i] = -1;
      if (out_waves) out_waves[i] = 0;
      if (out_match) out_match[i] = match;
      continue;
    }
    const PointResult r = predict_point(t, ci, b, m, nn, k, base_of(t, ci, k));
    out_lat[i] = r.lat;
    if (out_curve) out_curve[i] = ci;
    if (out_waves) out_waves[i] = uint32_t(r.waves);
    if (out_match) out_match[i] = match;
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
    if (c < 0 || c >= t.C || t.s_off[c + 1] <= t.s_off[c]) {
      out_lat[i] = __longlong_as_double(0x7FF8000000000000ll);
      if (out_waves) out_waves[i] = 0;
      continue;
    }
    const double base = base_of(t, c, s.w);
    const PointResult r = predict_point(t, c, s.x, s.y, s.z, s.w, base);
    out_lat[i] = r.lat;
    if (out_waves) out_waves[i] = uint32_t(r.waves);
    if (out_detail) {  // Prediction.components: base_us, new_throughput, wave_scale, blocks
      out_detail[4 * i] = base;
      out_detail[4 * i + 1] = interp_thr(t, c, __ull2double_rn(uint64_t(s.w)));
      out_detail[4 * i + 2] = wave_scale(t, c, r.waves);
      out_detail[4 * i + 3] = __ull2double_rn(r.blocks);
    }
  }
}

// --------------------------------------------------------------- membound
__global__ void membound_kernel(const double* __restrict__ f, const int32_t* __restrict__ mid,
                                int64_t n, const double* __restrict__ w,
                                const double* __restrict__ icpt, const double* __restrict__ floors,
                                int64_t n_models, double* __restrict__ out,
                                uint8_t* __restrict__ floored) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int mi = mid[i];
    if (mi < 0 || mi >= n_models) {
      out[i] = __longlong_as_double(0x7FF8000000000000ll);
      if (floored) floored[i] = 0;
      continue;
    }
    const double* x = f + 5 * i;
    const double* wm = w + 5 * mi;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 5; ++j) s = __fma_rn(wm[j], x[j], s);
    const double raw = __dadd_rn(s, icpt[mi]);
    const double fl = floors[mi];
    const bool below = raw < fl;
    out[i] = below ? fl : raw;
    if (floored) floored[i] = below ? 1 : 0;
  }
}

// ------------------------------------------------------------ exact fsum
// One warp per segment.  Terms are finite and >= 0.  Pass 1: max exponent E.
// Pass 2: every term whose bits all lie within a 4x64-bit window anchored at
// E is added EXACTLY as a fixed-point integer (integer adds are associative,
// so the warp tree reduction is exact); the 256-bit total is then rounded to
// nearest-even once.  A segment with a term below the window (dynamic range
// > ~180 bits) falls back to a sequential exact expansion sum on lane 0.
struct U256 {
  uint64_t w[4];
};

__device__ __forceinline__ void add256(U256& a, const U256& b) {
  asm("add.cc.u64 %0, %0, %4;\n\taddc.cc.u64 %1, %1, %5;\n\t"
      "addc.cc.u64 %2, %2, %6;\n\taddc.u64 %3, %3, %7;"
      : "+l"(a.w[0]), "+l"(a.w[1]), "+l"(a.w[2]), "+l"(a.w[3])
      : "l"(b.w[0]), "l"(b.w[1]), "l"(b.w[2]), "l"(b.w[3]));
}

__device__ double two_sum_fsum(const double* v, int64_t lo, int64_t hi) {
  // Shewchuk/msum (the algorithm behind math.fsum), partials kept in a
  // bounded local array; exact for non-negative finite inputs.
  double p[64];
  int np = 0;
  for (int64_t i = lo; i < hi; ++i) {
    double x = v[i];
    int j = 0;
    for (int q = 0; q < np; ++q) {
      double y = p[q];
      if (fabs(x) < fabs(y)) { double tmp = x; x = y; y = tmp; }
      const double hi_ = __dadd_rn(x, y);
      const double lo_ = __dsub_rn(y, __dsub_rn(hi_, x));
      if (lo_ != 0.0) p[j++] = lo_;
      x = hi_;
    }
    if (j < 64) p[j++] = x;
    np = j;
  }
  // sum partials from the top with the half-way correction of math.fsum
  if (np == 0) return 0.0;
  double hi_ = p[--np], lo_ = 0.0;
  while (np > 0) {
    const double x = hi_, y = p[--np];
    hi_ = __dadd_rn(x, y);
    const double yr = __dsub_rn(hi_, x);
    lo_ = __dsub_rn(y, yr);
    if (lo_ != 0.0) break;
  }
  if (np > 0 && ((lo_ < 0.0 && p[np - 1] < 0.0) || (lo_ > 0.0 && p[np - 1] > 0.0))) {
    const double y = __dmul_rn(lo_, 2.0);
    const double x = __dadd_rn(hi_, y);
    const double yr = __dsub_rn(x, hi_);
    if (y == yr) hi_ = x;
  }
  return hi_;
}

__global__ void segment_fsum_kernel(const double* __restrict__ v, const int64_t* __restrict__ off,
                                    int64_t nseg, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t seg = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (seg >= nseg) return;
  const int64_t lo = off[seg], hi = off[seg + 1];
  int emax = -2000;
  bool bad_nan = false, bad_inf = false, bad_neg = false;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    const double x = v[i];
    const uint64_t bits = uint64_t(__double_as_longlong(x));
    const int e = int((bits >> 52) & 0x7FF);
    if (x != x) bad_nan = true;
    else if (e == 0x7FF) bad_inf = true;
    else if (bits >> 63 && x != 0.0) bad_neg = true;
    else if (x != 0.0) emax = max(emax, e == 0 ? 1 : e);
  }
  for (int o = 16; o; o >>= 1) emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
  bad_nan = __any_sync(0xFFFFFFFFu, bad_nan);
  bad_inf = __any_sync(0xFFFFFFFFu, bad_inf);
  bad_neg = __any_sync(0xFFFFFFFFu, bad_neg);
  if (bad_nan || bad_neg || bad_inf) {
    if (lane == 0)
      out[seg] = (bad_nan || bad_neg) ? __longlong_as_double(0x7FF8000000000000ll)
                                      : __longlong_as_double(0x7FF0000000000000ll);
    return;
  }
  if (emax == -2000) {  // empty or all zeros
    if (lane == 0) out[seg] = 0.0;
    return;
  }
  // window: LSB weight 2^(emax - 1075 - 180); term with biased exponent e
  // (e==0 -> subnormal, scale as e=1) contributes mant << (e - emax + 180).
  constexpr int kGuard = 180;
  U256 acc = {{0, 0, 0, 0}};
  bool below = false;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    const uint64_t bits = uint64_t(__double_as_longlong(v[i]));
    if (bits == 0) continue;
    const int be = int((bits >> 52) & 0x7FF);
    const uint64_t mant = (bits & 0xFFFFFFFFFFFFFull) | (be ? (1ull << 52) : 0ull);
    const int e = be ? be : 1;
    const int sh = e - emax + kGuard;
    if (sh < 0) { below = true; continue; }
    U256 term = {{0, 0, 0, 0}};
    const int limb = sh >> 6, bit = sh & 63;
    term.w[limb] = mant << bit;
    if (bit && limb + 1 < 4) term.w[limb + 1] = mant >> (64 - bit);
    add256(acc, term);
  }
  below = __any_sync(0xFFFFFFFFu, below);
  if (below) {
    if (lane == 0) out[seg] = two_sum_fsum(v, lo, hi);
    return;
  }
  for (int o = 16; o; o >>= 1) {
    U256 other;
    for (int q = 0; q < 4; ++q) other.w[q] = __shfl_xor_sync(0xFFFFFFFFu, acc.w[q], o);
    add256(acc, other);
  }
  if (lane != 0) return;
  // round the exact 256-bit integer to 53 bits, nearest-even
  int top = 255;
  while (top >= 0 && !((acc.w[top >> 6] >> (top & 63)) & 1ull)) --top;
  auto bit_at = [&](int p) -> uint64_t { return p < 0 ? 0 : (acc.w[p >> 6] >> (p & 63)) & 1ull; };
  uint64_t mant = 0;
  int shift = 0;  // value = mant * 2^shift * LSB
  if (top < 53) {
    mant = acc.w[0];  // fewer than 54 significant bits: exact
  } else {
    for (int p = top; p > top - 53; --p) mant = (mant << 1) | bit_at(p);
    shift = top - 52;
    const uint64_t guard = bit_at(top - 53);
    bool sticky = false;
    for (int w = 0; w < 4 && !sticky; ++w) {
      const int lo_bit = w * 64, hi_bit = min(w * 64 + 63, top - 54);
      if (hi_bit < lo_bit) break;
      const int nbits = hi_bit - lo_bit + 1;
      const uint64_t msk = nbits >= 64 ? ~0ull : ((1ull << nbits) - 1ull);
      sticky = (acc.w[w] & msk) != 0;
    }
    if (guard && (sticky || (mant & 1ull))) {
      mant += 1;
      if (mant >> 53) { mant >>= 1; shift += 1; }
    }
  }
  // LSB weight exponent: (emax - 1075) - kGuard  (unbiased exponent of 1 ulp
  // at biased exponent emax is emax - 1075)
  const int exp2 = shift + (emax - 1075) - kGuard;
  out[seg] = scalbn(double(mant), exp2);
}

__global__ void nan_scan_kernel(const double* __restrict__ v, int64_t n,
                                unsigned long long* __restrict__ first) {
  unsigned long long mine = ~0ull;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    if (v[i] != v[i]) { mine = (unsigned long long)i; break; }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xFFFFFFFFu, mine, o);
    mine = x < mine ? x : mine;
  }
  if ((threadIdx.x & 31) == 0 && mine != ~0ull) atomicMin(first, mine);
}

GridLaunch plan_grid(const TablesDev& t, const GridDev& g, bool all_curves) {
  GridLaunch gl{};
  const int64_t rows = g.nM * g.nN;
  const int64_t nb = g.b_hi - g.b_lo;
  const int64_t target = 148 * 8;
  gl.kpt = 4;
  auto ktiles_for = [&](int kpt) { return (g.nK + int64_t(kpt) * kThreads - 1) / (int64_t(kpt) * kThreads); };
  gl.ktiles = int(ktiles_for(gl.kpt));
  while (gl.kpt > 1 && rows * gl.ktiles < target) {
    gl.kpt >>= 1;
    gl.ktiles = int(ktiles_for(gl.kpt));
  }
  int64_t ctas = rows * gl.ktiles;
  gl.nbs = 1;
  if (ctas < target && nb > 1) gl.nbs = int(std::min<int64_t>(nb, (target + ctas - 1) / ctas));
  gl.bper = (nb + gl.nbs - 1) / gl.nbs;
  gl.nbs = int((nb + gl.bper - 1) / gl.bper);
  if (all_curves) {
    gl.mode = (t.all_gemm && 8ll * t.C * (gl.bper + 1) <= 96 * 1024) ? 0 : 2;
    gl.smem = gl.mode == 0 ? ((8ll * t.C + 15) & ~15ll) + 8ll * t.C * gl.bper : 0;
    return gl;
  }
  if (!t.all_gemm) gl.mode = 2;
  else if (8ll * t.C * gl.bper <= 48 * 1024 && t.C <= 4 * g.nK) gl.mode = 0;
  else gl.mode = 1;
  gl.smem = smem_layout(t.R, t.G, t.C, gl.bper, gl.mode).total;
  return gl;
}

}  // namespace

int64_t grid_workspace_elems(const TablesDev& t, const GridDev& g) {
  const int64_t e = int64_t(t.C) * g.nK;
  return e <= (int64_t(1) << 25) ? e : 0;  // base table only when <= 256 MiB
}

template <bool V, int M>
static cudaError_t launch_grid_t(const TablesDev& t, const GridDev& g, const GridLaunch& gl,
                                 const double* base, const LaunchOut& out, cudaStream_t s) {
  auto* fn = t.G <= 32 ? grid_kernel<V, M, true> : grid_kernel<V, M, false>;
  if (gl.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gl.smem));
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = g.nM * g.nN * gl.ktiles * int64_t(gl.nbs);
  if (blocks > 0) fn<<<unsigned(blocks), kThreads, gl.smem, s>>>(t, g, gl, base, out);
  return cudaGetLastError();
}

int launch_grid(const TablesDev& t, const GridDev& g, int64_t /*max_group*/, double* ws,
                int64_t ws_elems, const LaunchOut& out, void* stream, int stages) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t card = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  if (card == 0) return 0;
  const GridLaunch gl = plan_grid(t, g, false);
  if (gl.smem > 227 * 1024) return int(cudaErrorInvalidValue);
  const double* base = nullptr;
  if (ws && ws_elems >= int64_t(t.C) * g.nK && t.C > 0) {
    const int64_t total = int64_t(t.C) * g.nK;
    const int nb = int(std::min<int64_t>((total + 255) / 256, 148 * 16));
    if (stages & kStageBase) base_table_kernel<<<nb, 256, 0, s>>>(t, g.K, g.nK, ws);
    base = ws;
  }
  const bool v = out.curve != nullptr;
  cudaError_t e = cudaSuccess;
  if (!(stages & kStageGrid)) {
  } else if (v) {
    e = gl.mode == 0 ? launch_grid_t<true, 0>(t, g, gl, base, out, s)
        : gl.mode == 1 ? launch_grid_t<true, 1>(t, g, gl, base, out, s)
                       : launch_grid_t<true, 2>(t, g, gl, base, out, s);
  } else {
    e = gl.mode == 0 ? launch_grid_t<false, 0>(t, g, gl, base, out, s)
        : gl.mode == 1 ? launch_grid_t<false, 1>(t, g, gl, base, out, s)
                       : launch_grid_t<false, 2>(t, g, gl, base, out, s);
  }
  if (e != cudaSuccess) return int(e);
  if (g.n_fix > 0 && (stages & kStageFixup)) {
    const int nb = int((g.n_fix + 127) / 128);
    if (v) fixup_kernel<true><<<nb, 128, 0, s>>>(t, g, out);
    else fixup_kernel<false><<<nb, 128, 0, s>>>(t, g, out);
  }
  return int(cudaGetLastError());
}

int launch_grid_all_curves(const TablesDev& t, const GridDev& g, double* ws, double* out,
                           void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t card = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  if (card == 0 || t.C == 0) return 0;
  const GridLaunch gl = plan_grid(t, g, true);
  const int64_t total = int64_t(t.C) * g.nK;
  const int nb = int(std::min<int64_t>((total + 255) / 256, 148 * 16));
  base_table_kernel<<<nb, 256, 0, s>>>(t, g.K, g.nK, ws);
  if (gl.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(all_curves_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(gl.smem));
    if (e != cudaSuccess) return int(e);
  }
  const int64_t blocks = g.nM * g.nN * gl.ktiles * int64_t(gl.nbs);
  all_curves_kernel<<<unsigned(blocks), kThreads, gl.smem, s>>>(t, g, gl, ws, out);
  return int(cudaGetLastError());
}

int launch_points(const TablesDev& t, const uint32_t* shapes, int64_t n, const double* lut,
                  int64_t lut_n, double* out_lat, int32_t* out_curve, uint32_t* out_waves,
                  int8_t* out_match, int32_t* out_record, double* out_dist, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t smem = 20ll * t.R + 16;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(points_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return int(e);
  }
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 8));
  points_kernel<<<nb, kThreads, smem, s>>>(t, reinterpret_cast<const uint4*>(shapes), n, lut,
                                          lut_n, out_lat, out_curve, out_waves, out_match,
                                          out_record, out_dist);
  return int(cudaGetLastError());
}

int launch_points_curve(const TablesDev& t, const uint32_t* shapes, const int32_t* curves, int64_t n,
                        double* out_lat, uint32_t* out_waves, double* out_detail, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 16));
  points_curve_kernel<<<nb, kThreads, 0, s>>>(t, reinterpret_cast<const uint4*>(shapes), curves, n,
                                             out_lat, out_waves, out_detail);
  return int(cudaGetLastError());
}

int launch_membound(const double* f, const int32_t* mid, int64_t n, const double* w,
                    const double* b, const double* floors, int64_t n_models, double* out,
                    uint8_t* floored, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 16));
  membound_kernel<<<nb, kThreads, 0, s>>>(f, mid, n, w, b, floors, n_models, out, floored);
  return int(cudaGetLastError());
}

int launch_nan_scan(const double* v, int64_t n, unsigned long long* first, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
  nan_scan_kernel<<<nb, 256, 0, s>>>(v, n, first);
  return int(cudaGetLastError());
}

int launch_segment_fsum(const double* v, const int64_t* off, int64_t nseg, double* out,
                        void* stream) {
  if (nseg == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t threads = nseg * 32;
  const int nb = int((threads + 255) / 256);
  segment_fsum_kernel<<<nb, 256, 0, s>>>(v, off, nseg, out);
  return int(cudaGetLastError());
}

}  // namespace pm2l
