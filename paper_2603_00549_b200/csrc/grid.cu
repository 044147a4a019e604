// Grid mode: the canonical (batch, m, n, k) sweep of predict_grid_slice
// (pm2lat/_kernels.pyx:76-133, backend.py:49-88), plus "mode X" (every
// candidate kernel per shape) and the unresolved-point scan.
//
// Per launch (all device-side, CUDA-graph capturable):
//   base_table_kernel  base(c, k) = ref_dur*(k/ref_dim)*(ref_thr/thr(c,k)) for
//                      every curve and k value (per-curve samples in smem);
//                      releases the dependent grid kernel immediately
//                      (programmatic dependent launch)
//   grid_kernel        one CTA per ((m, n) row, k tile, batch slab).  Setup
//                      overlaps the base-table kernel: warp 0 builds the
//                      member-class staircases of D_j = max(|lm_j-qm|,|ln_j-qn|)
//                      (warp scan + ballot) while the other warps build
//                      Tmn[c] = ceil(m/tm)*ceil(n/tn)*sk and the wave-scale
//                      table W[c][ib] in shared memory; after
//                      griddepcontrol.wait each thread owns k values: nearest
//                      config by the outward k-group sweep, then one DMUL and
//                      one coalesced 8-byte store per batch value
//   fixup_kernel       exact-record hits (take priority over nearest)
#include <algorithm>

#include "common.cuh"

namespace pm2l {
namespace {

using namespace dev;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;"); }

// ----------------------------------------------------------- base table
// base[c][ik] for every curve c and k value; one CTA per (curve, k chunk)
// with the curve's samples staged in shared memory.
constexpr int kMaxSmemSamples = 256;

__global__ void __launch_bounds__(256) base_table_kernel(TablesDev t, const uint64_t* __restrict__ K,
                                                         int nK, double* __restrict__ base) {
  pdl_release();  // the grid kernel may start its (independent) row setup now
  __shared__ double sd[kMaxSmemSamples], sy[kMaxSmemSamples];
  const int c = blockIdx.y;
  const int lo = t.s_off[c], hi = t.s_off[c + 1], ns = hi - lo;
  if (ns <= 0) {
    for (int ik = blockIdx.x * blockDim.x + threadIdx.x; ik < nK; ik += gridDim.x * blockDim.x)
      base[int64_t(c) * nK + ik] = 0.0;
    return;
  }
  const bool staged = ns <= kMaxSmemSamples;
  if (staged) {
    for (int j = threadIdx.x; j < ns; j += blockDim.x) {
      sd[j] = t.s_dims[lo + j];
      sy[j] = t.s_thrs[lo + j];
    }
  }
  __syncthreads();
  for (int ik = blockIdx.x * blockDim.x + threadIdx.x; ik < nK; ik += gridDim.x * blockDim.x) {
    const double nd = __ull2double_rn(K[ik]);
    const double thr = staged ? interp_samples(sd, sy, 0, ns, nd)
                              : interp_samples(t.s_dims, t.s_thrs, lo, hi, nd);
    base[int64_t(c) * nK + ik] = base_from_thr(t, c, nd, thr);
  }
}

// ------------------------------------------------------------ grid kernel
struct GridLaunch {
  int kpt;       // k values per thread
  int ktiles;    // k tiles per row  (gridDim.y)
  int nbs;       // batch slabs      (gridDim.z)
  int bper;      // batch values per slab
  int mode;      // 0: GEMM + W table, 1: GEMM per point, 2: general (row-block)
  int near;      // 0: general sweep, 1: sweep + tie mask (G <= 32), 2: one member class
  // grid_kernel shared-memory layout (byte offsets), computed on the host
  int off_sD, off_sP, off_cls, off_T, off_W, off_gcur, off_gst, off_glk;
  int64_t smem;
};

struct ClassRow {
  uint64_t dmin;    // min over the class members of D (ordered bits)
  int32_t lastpos;  // member position attaining dmin first
  int32_t len;      // staircase length
};

void smem_layout(const TablesDev& t, GridLaunch& gl) {
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = (o + bytes + 15) & ~int64_t(15);
    return int(at);
  };
  gl.off_sD = take(8ll * t.CM);
  gl.off_sP = take(4ll * t.CM);
  gl.off_cls = take(16ll * t.NC);
  gl.off_T = take(gl.mode <= 1 ? 8ll * t.C : 0);
  gl.off_W = take(gl.mode == 0 ? 8ll * t.C * gl.bper : 0);
  gl.off_gcur = take(4ll * t.R);
  gl.off_gst = take(4ll * t.G);
  gl.off_glk = take(8ll * t.G);
  gl.smem = o;
}

struct RowView {
  const ClassRow* cls;
  const uint64_t* sD;
  const int32_t* sP;
};

// Scan index of the first member of group g whose distance equals `best`
// (the group attains best): the first staircase entry with D <= best.

__device__ __forceinline__ int group_index(const TablesDev& t, const RowView& rv, int g,
                                           uint64_t best) {
  const int c = t.grp_class[g];
  const ClassRow cr = rv.cls[c];
  int pos = cr.lastpos;
  if (best != cr.dmin) {
    int s = t.cls_start[c];
    while (rv.sD[s] > best) ++s;
    pos = rv.sP[s];
  }
  return t.g_idx[t.grp_start[g] + pos];
}

// Nearest-config argmin for one query k (_kernels.pyx:29-47 semantics).
// dist(i) = max(D_i, dk_g(i)), dk_g = |lk_g - qk|.  Groups are sorted by lk,
// so dk_g grows monotonically (IEEE subtraction is monotone) moving away from
// qk's insertion point: sweep right then left, stopping a side as soon as
// dk_g exceeds the running best.  Ties (equal distance) resolve to the
// smallest scan index among every member attaining the final best.
// Returns the ORIGINAL candidate scan index (INT32_MAX when G == 0).
template <bool G32>
__device__ __forceinline__ int nearest_sweep(const TablesDev& t, const RowView& rv,
                                             const double* __restrict__ glk, double qk,
                                             int start) {
  uint64_t best = ~0ull;
  uint32_t mask = 0;
  int best_i = 0x7FFFFFFF;
  auto visit = [&](int g) -> bool {
    const uint64_t dk = abs_bits(__dsub_rn(glk[g], qk));
    if (dk > best) return false;
    const uint64_t dg = umax64(dk, rv.cls[t.grp_class[g]].dmin);
    if (G32) {
      if (dg < best) { best = dg; mask = 1u << g; }
      else if (dg == best) mask |= 1u << g;
    } else if (dg <= best) {
      const int idx = group_index(t, rv, g, dg);
      if (dg < best || idx < best_i) best_i = idx;
      best = dg;
    }
    return true;
  };
  for (int g = start; g < t.G; ++g)
    if (!visit(g)) break;
  for (int g = start - 1; g >= 0; --g)
    if (!visit(g)) break;
  if (G32) {
    while (mask) {
      const int g = __ffs(mask) - 1;
      mask &= mask - 1;
      const int idx = group_index(t, rv, g, best);
      best_i = idx < best_i ? idx : best_i;
    }
  }
  return best_i;
}

// One member class (every kernel recorded at every sample k — the shipped
// presets): all groups share D, dmin and the staircase, and between tied
// groups the one with the smaller lk has the smaller scan index (same (m, n)
// at the same member position, then k decides; host-verified: coordinates
// < 2^44 so equal logs imply equal coordinates).  Hence
//   best = max(dmin, min(dk_left, dk_right))   (nearest groups to qk)
//   winner = the leftmost group attaining best, member = staircase(best).
// Returns (group, member position).
__device__ __forceinline__ int2 nearest_one_class(int G, const double* __restrict__ glk,
                                                  const RowView& rv, uint64_t dmin, int lastpos,
                                                  double qk, int start) {
  auto dk = [&](int g) { return abs_bits(__dsub_rn(glk[g], qk)); };
  const uint64_t dkL = start > 0 ? dk(start - 1) : ~0ull;
  const uint64_t dkR = start < G ? dk(start) : ~0ull;
  const uint64_t mn = dkL < dkR ? dkL : dkR;
  int g, pos;
  if (mn <= dmin) {            // best == dmin: every group with dk <= dmin ties
    if (dkL <= dmin) {
      g = start - 1;
      while (g > 0 && dk(g - 1) <= dmin) --g;
    } else {
      g = start;
    }
    pos = lastpos;
  } else {                     // best == mn > dmin
    if (dkL == mn) {
      g = start - 1;
      while (g > 0 && dk(g - 1) == mn) --g;
    } else {
      g = start;
    }
    int s = 0;
    while (rv.sD[s] > mn) ++s;
    pos = rv.sP[s];
  }
  return make_int2(g, pos);
}

constexpr int kGridThreads = 128;

template <bool VERIFY, int MODE, int NEAR, int NB>
__global__ void __launch_bounds__(kGridThreads, 8) grid_kernel(TablesDev t, GridDev g, GridLaunch gl,
                                                        const double* __restrict__ base_tab,
                                                        LaunchOut out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* sD = reinterpret_cast<uint64_t*>(smem + gl.off_sD);
  int32_t* sP = reinterpret_cast<int32_t*>(smem + gl.off_sP);
  ClassRow* scls = reinterpret_cast<ClassRow*>(smem + gl.off_cls);
  uint64_t* T = reinterpret_cast<uint64_t*>(smem + gl.off_T);
  double* W = reinterpret_cast<double*>(smem + gl.off_W);
  int32_t* gcur = reinterpret_cast<int32_t*>(smem + gl.off_gcur);
  int32_t* gst = reinterpret_cast<int32_t*>(smem + gl.off_gst);
  double* glk = reinterpret_cast<double*>(smem + gl.off_glk);

  const int row = blockIdx.x;
  const int nN = int(g.nN), nK = int(g.nK);
  const int im = row / nN, jn = row - im * nN;
  const int ib0 = int(blockIdx.z) * gl.bper;  // slice-relative
  const int nb = min(int(g.b_hi - g.b_lo), ib0 + gl.bper) - ib0;
  const int tid = threadIdx.x;
  const uint64_t m = g.M[im], n = g.N[jn];

  // ---- row setup (independent of the base table: overlaps its kernel)
  if (tid < 32) {
    // member-class staircases: prefix minimum of D in member (scan) order
    const int lane = tid;
    const double qm = g.logM[im], qn = g.logN[jn];
    for (int ci = 0; ci < t.NC; ++ci) {
      const int start = t.cls_start[ci], size = t.cls_size[ci];
      uint64_t carry = ~0ull;
      int len = 0, lastpos = 0;
      for (int b0 = 0; b0 < size; b0 += 32) {
        const int j = b0 + lane;
        const uint64_t d = j < size ? umax64(abs_bits(__dsub_rn(t.cls_lm[start + j], qm)),
                                             abs_bits(__dsub_rn(t.cls_ln[start + j], qn)))
                                    : ~0ull;
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
          sP[pos] = j;
        }
        if (mask) lastpos = b0 + 31 - __clz(mask);
        len += __popc(mask);
        const uint64_t tail = __shfl_sync(0xFFFFFFFFu, pm, 31);
        if (tail < carry) carry = tail;
      }
      if (lane == 0) scls[ci] = ClassRow{carry, lastpos, len};
    }
  } else {
    // tiles per (m, n) and the curve-major wave-scale table W[c][ib]
    const int nth = blockDim.x - 32, me = tid - 32;
    if (MODE <= 1) {
      for (int c = me; c < t.C; c += nth) {
        if (!curve_valid(t, c)) continue;
        const uint64_t tmn = ceil_div_c(t, c, 0, m, t.tile_m[c]) *
                             ceil_div_c(t, c, 1, n, t.tile_n[c]) * t.split_k[c];
        T[c] = tmn;
        if (MODE == 0) {
          const uint64_t bpw = t.bpw[c];
          for (int ib = 0; ib < nb; ++ib)
            W[c * nb + ib] =
                wave_scale(t, c, ceil_div_c(t, c, 2, g.B[g.b_lo + ib0 + ib] * tmn, bpw));
        }
      }
    }
    for (int j = me; j < t.R; j += nth) gcur[j] = t.g_curve[j];
    for (int j = me; j < t.G; j += nth) {
      gst[j] = t.grp_start[j];
      glk[j] = t.grp_lk[j];
    }
  }
  __syncthreads();
  const RowView rv{scls, sD, sP};
  uint64_t dmin1 = 0;
  int lastpos1 = 0;
  if (NEAR == 2) {
    dmin1 = scls[0].dmin;
    lastpos1 = scls[0].lastpos;
  }
  pdl_wait();  // base table complete and visible

  // ---- points: thread owns kpt k values (stride blockDim); every batch value
  const int64_t plane = g.nM * g.nN * g.nK;
  double* const obase = out.lat + int64_t(ib0) * plane + int64_t(row) * nK;
  const int k0 = int(blockIdx.y) * gl.kpt * int(blockDim.x);
  if (NEAR == 2 && MODE == 0 && !VERIFY && NB > 0) {
    // hot path, software-pipelined in groups of U k values: all kinfo loads,
    // then all nearest searches, then all base-table loads in flight
    // together, then the stores (memory-level parallelism for a kernel whose
    // per-point chain is kinfo -> curve -> base -> store)
    constexpr int U = 4;
    const int step = int(blockDim.x);
    for (int j0 = 0; j0 < gl.kpt; j0 += U) {
      double2 ki[U];
      int ik[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ik[u] = k0 + (j0 + u) * step + tid;
        ki[u] = ik[u] < nK ? *reinterpret_cast<const double2*>(&g.kinfo[ik[u]])
                           : make_double2(0.0, 0.0);
      }
      int ci[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ik[u] < nK && j0 + u < gl.kpt) {
          const int2 gp = nearest_one_class(t.G, glk, rv, dmin1, lastpos1, ki[u].x,
                                            __double2loint(ki[u].y));
          ci[u] = gcur[gst[gp.x] + gp.y];
        } else {
          ci[u] = -2;  // out of range
        }
      }
      double bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) bv[u] = ci[u] >= 0 ? base_tab[ci[u] * nK + ik[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ci[u] == -2) continue;
        double* o = obase + ik[u];
        if (ci[u] < 0) {
          if (out.nan_stats) {
            atomicMin(out.nan_stats, (unsigned long long)(o - out.lat));
            atomicAdd(out.nan_stats + 1, (unsigned long long)NB);
          }
#pragma unroll
          for (int ib = 0; ib < NB; ++ib) o[ib * plane] = qnan();
          continue;
        }
        const double* w = W + ci[u] * NB;
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) o[ib * plane] = __dmul_rn(bv[u], w[ib]);
      }
    }
    return;
  }
  for (int j = 0; j < gl.kpt; ++j) {
    const int ik = k0 + j * int(blockDim.x) + tid;
    if (ik >= nK) break;
    const double2 ki = *reinterpret_cast<const double2*>(&g.kinfo[ik]);
    const int start = __double2loint(ki.y);
    int ci;
    if (NEAR == 2) {
      const int2 gp = nearest_one_class(t.G, glk, rv, dmin1, lastpos1, ki.x, start);
      ci = gcur[gst[gp.x] + gp.y];
    } else {
      const int best = nearest_sweep<NEAR == 1>(t, rv, glk, ki.x, start);
      ci = best < t.R ? t.cand_curve[best] : -1;
    }
    double* o = obase + ik;
    if (ci < 0) {
      if (out.nan_stats) {
        atomicMin(out.nan_stats, (unsigned long long)(o - out.lat));
        atomicAdd(out.nan_stats + 1, (unsigned long long)nb);
      }
      for (int ib = 0; ib < nb; ++ib, o += plane) {
        *o = qnan();
        if (VERIFY) {
          const int64_t p = o - out.lat;
          out.curve[p] = -1;
          out.blocks[p] = 0;
          out.waves[p] = 0;
        }
      }
      continue;
    }
    const double base = base_tab ? base_tab[ci * nK + ik] : base_of(t, ci, g.K[ik]);
    if (MODE == 0 && !VERIFY) {
      const double* w = W + ci * nb;
      if (NB > 0) {
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) o[ib * plane] = __dmul_rn(base, w[ib]);
      } else {
        for (int ib = 0; ib < nb; ++ib, o += plane) *o = __dmul_rn(base, w[ib]);
      }
      continue;
    }
    const uint64_t k = g.K[ik];
    for (int ib = 0; ib < nb; ++ib, o += plane) {
      const uint64_t b = g.B[g.b_lo + ib0 + ib];
      double lat;
      uint64_t blocks, waves;
      if (MODE <= 1) {
        blocks = b * T[ci];
        waves = ceil_div_c(t, ci, 2, blocks, t.bpw[ci]);
        lat = __dmul_rn(base, wave_scale(t, ci, waves));
      } else {
        const PointResult r = predict_point(t, ci, b, m, n, k, base);
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

// Exact-record hits take priority over the nearest result (_kernels.pyx:107-110).
template <bool VERIFY>
__global__ void fixup_kernel(TablesDev t, GridDev g, LaunchOut out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= g.n_fix) return;
  const int64_t p = g.fix_pos[i];
  const uint64_t* c4 = g.fix_coord + 4 * i;
  const int ci = g.fix_curve[i];
  if (out.nan_stats) {
    // the grid kernel counted this point by its nearest result; re-count it
    // by its exact result.  A NaN that disappears may have been the minimum:
    // flag the stats dirty so the caller re-derives it (pm2l_nan_scan).
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
    out.lat[p] = qnan();
    if (VERIFY) { out.curve[p] = -1; out.blocks[p] = 0; out.waves[p] = 0; }
    return;
  }
  const PointResult r = predict_point(t, ci, c4[0], c4[1], c4[2], c4[3], base_of(t, ci, c4[3]));
  out.lat[p] = r.lat;
  if (VERIFY) { out.curve[p] = ci; out.blocks[p] = r.blocks; out.waves[p] = r.waves; }
}

// ------------------------------------------------------- mode X (all curves)
__global__ void __launch_bounds__(kThreads) all_curves_kernel(TablesDev t, GridDev g, GridLaunch gl,
                                                              const double* __restrict__ base_tab,
                                                              double* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* Tmn = reinterpret_cast<uint64_t*>(smem);
  double* W = reinterpret_cast<double*>(smem + ((8ll * t.C + 15) & ~15ll));
  const int row = blockIdx.x;
  const int nN = int(g.nN), nK = int(g.nK);
  const int im = row / nN, jn = row - im * nN;
  const int ib0 = int(g.b_lo) + int(blockIdx.z) * gl.bper;
  const int ib1 = min(int(g.b_hi), ib0 + gl.bper);
  if (ib0 >= ib1) return;
  const int nb = ib1 - ib0;
  const uint64_t m = g.M[im], n = g.N[jn];
  const int tid = threadIdx.x;
  const bool table = gl.mode == 0;
  if (table) {
    for (int c = tid; c < t.C; c += blockDim.x)
      Tmn[c] = curve_valid(t, c) ? ceil_div_c(t, c, 0, m, t.tile_m[c]) *
                                       ceil_div_c(t, c, 1, n, t.tile_n[c]) * t.split_k[c]
                                 : 0;
    __syncthreads();
    for (int e = tid; e < nb * t.C; e += blockDim.x) {
      const int ib = e / t.C;
      const int c = e - ib * t.C;
      if (curve_valid(t, c))
        W[e] = wave_scale(t, c, ceil_div_c(t, c, 2, g.B[ib0 + ib] * Tmn[c], t.bpw[c]));
    }
    __syncthreads();
  }
  const int64_t slice = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  const int64_t plane = g.nM * g.nN * g.nK;
  const int64_t row_off = int64_t(ib0 - g.b_lo) * plane + int64_t(row) * nK;
  const int k0 = int(blockIdx.y) * gl.kpt * int(blockDim.x);
  for (int j = 0; j < gl.kpt; ++j) {
    const int ik = k0 + j * int(blockDim.x) + tid;
    if (ik >= nK) break;
    const uint64_t k = g.K[ik];
    for (int c = 0; c < t.C; ++c) {
      const double base = base_tab[int64_t(c) * nK + ik];
      const bool valid = curve_valid(t, c);
      double* o = out + int64_t(c) * slice + row_off + ik;
      for (int ib = 0; ib < nb; ++ib, o += plane) {
        double lat;
        if (!valid) lat = qnan();
        else if (table) lat = __dmul_rn(base, W[ib * t.C + c]);
        else lat = predict_point(t, c, g.B[ib0 + ib], m, n, k, base).lat;
        __stcs(o, lat);
      }
    }
  }
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
  const int threads = all_curves ? kThreads : kGridThreads;
  auto ktiles_for = [&](int kpt) {
    return int((g.nK + int64_t(kpt) * threads - 1) / (int64_t(kpt) * threads));
  };
  gl.kpt = all_curves ? 4 : 8;
  gl.ktiles = ktiles_for(gl.kpt);
  while (gl.kpt > 1 && rows * gl.ktiles < target) {
    gl.kpt >>= 1;
    gl.ktiles = ktiles_for(gl.kpt);
  }
  const int64_t ctas = rows * gl.ktiles;
  int64_t nbs = 1;
  if (ctas < target && nb > 1) nbs = std::min<int64_t>(nb, (target + ctas - 1) / ctas);
  gl.bper = int((nb + nbs - 1) / nbs);
  gl.nbs = int((nb + gl.bper - 1) / gl.bper);
  if (all_curves) {
    gl.mode = (t.all_gemm && 8ll * t.C * (gl.bper + 1) <= 96 * 1024) ? 0 : 2;
    return gl;
  }
  gl.mode = t.all_gemm ? 0 : 2;
  gl.near = (t.NC == 1 && t.lowest_wins) ? 2 : (t.G <= 32 ? 1 : 0);
  smem_layout(t, gl);
  if (gl.mode == 0 && gl.smem > 160 * 1024) {  // W slice too large for smem
    gl.mode = 1;
    smem_layout(t, gl);
  }
  return gl;
}

bool grid_dims_ok(const GridDev& g, const GridLaunch& gl) {
  return g.nM * g.nN <= 0x7FFFFFFFll && gl.ktiles <= 65535 && gl.nbs <= 65535 &&
         g.nK <= 0x3FFFFFFFll && g.nB <= 0x7FFFFFFFll;
}

template <bool V, int M>
cudaError_t launch_grid_t(const TablesDev& t, const GridDev& g, const GridLaunch& gl,
                          const double* base, const LaunchOut& out, cudaStream_t s) {
  const bool nb4 = M == 0 && !V && gl.bper == 4 && (g.b_hi - g.b_lo) % 4 == 0;
  auto* fn = gl.near == 2 ? (nb4 ? grid_kernel<V, M, 2, 4> : grid_kernel<V, M, 2, 0>)
             : gl.near == 1 ? grid_kernel<V, M, 1, 0>
                            : grid_kernel<V, M, 0, 0>;
  if (gl.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gl.smem));
    if (e != cudaSuccess) return e;
  }
  // programmatic dependent launch: the row setup overlaps the base-table
  // kernel; griddepcontrol.wait guards the first base-table read
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(g.nM * g.nN), unsigned(gl.ktiles), unsigned(gl.nbs));
  cfg.blockDim = dim3(kGridThreads);
  cfg.dynamicSmemBytes = size_t(gl.smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, t, g, gl, base, out);
}

void launch_base_table(const TablesDev& t, const GridDev& g, double* ws, cudaStream_t s) {
  const int chunks = int(std::min<int64_t>((g.nK + 255) / 256, 64));
  base_table_kernel<<<dim3(chunks, t.C), 256, 0, s>>>(t, g.K, int(g.nK), ws);
}

}  // namespace

int64_t grid_workspace_elems(const TablesDev& t, const GridDev& g) {
  return int64_t(t.C) * g.nK;
}

int launch_grid(const TablesDev& t, const GridDev& g, int64_t /*max_group*/, double* ws,
                int64_t ws_elems, const LaunchOut& out, void* stream, int stages) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t card = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  if (card == 0) return 0;
  const GridLaunch gl = plan_grid(t, g, false);
  const int64_t need = int64_t(t.C) * g.nK;
  if ((need > 0 && (!ws || ws_elems < need)) || !grid_dims_ok(g, gl) || gl.smem > 227 * 1024 ||
      t.C > 65535 || need > 0x7FFFFFFFll)
    return int(cudaErrorInvalidValue);
  const double* base = t.C > 0 ? ws : nullptr;
  if ((stages & kStageBase) && t.C > 0) launch_base_table(t, g, ws, s);
  const bool v = out.curve != nullptr;
  cudaError_t e = cudaSuccess;
  if (stages & kStageGrid) {
    if (v) {
      e = gl.mode == 0 ? launch_grid_t<true, 0>(t, g, gl, base, out, s)
          : gl.mode == 1 ? launch_grid_t<true, 1>(t, g, gl, base, out, s)
                         : launch_grid_t<true, 2>(t, g, gl, base, out, s);
    } else {
      e = gl.mode == 0 ? launch_grid_t<false, 0>(t, g, gl, base, out, s)
          : gl.mode == 1 ? launch_grid_t<false, 1>(t, g, gl, base, out, s)
                         : launch_grid_t<false, 2>(t, g, gl, base, out, s);
    }
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
  GridLaunch gl = plan_grid(t, g, true);
  if (!grid_dims_ok(g, gl) || t.C > 65535) return int(cudaErrorInvalidValue);
  launch_base_table(t, g, ws, s);
  const int64_t smem = gl.mode == 0 ? ((8ll * t.C + 15) & ~15ll) + 8ll * t.C * gl.bper : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(all_curves_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return int(e);
  }
  const dim3 grid(unsigned(g.nM * g.nN), unsigned(gl.ktiles), unsigned(gl.nbs));
  all_curves_kernel<<<grid, kThreads, smem, s>>>(t, g, gl, ws, out);
  return int(cudaGetLastError());
}

int launch_nan_scan(const double* v, int64_t n, unsigned long long* first, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
  nan_scan_kernel<<<nb, 256, 0, s>>>(v, n, first);
  return int(cudaGetLastError());
}

}  // namespace pm2l
