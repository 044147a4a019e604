// General grid kernel (pm2lat/_kernels.pyx:76-133): warp-specialised
// per-k k-group sweep.  Covers several member classes, row-block families,
// the verification outputs (curve, blocks, waves) and odd k axes.
#include "grid_common.cuh"

namespace pm2l {
namespace gk {
namespace {

struct ClassRow {
  uint64_t dmin;    // min over the class members of D (ordered bits)
  int32_t lastpos;  // member position attaining dmin first
  int32_t len;      // staircase length
};

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
constexpr int kBarFull = 1;   // ids 1, 2
constexpr int kBarEmpty = 3;  // ids 3, 4

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

// Row state of one (row, slab) tile, produced into buffer `buf`.
// Row scalars a producer needs, loaded one tile ahead (latency off the
// producer's critical path).
struct RowPre {
  double qm, qn;
  uint64_t m, n;
};

__device__ __forceinline__ RowPre load_row(const GridDev& g, int row) {
  const int nN = int(g.nN);
  const int im = row / nN, jn = row - im * nN;
  return RowPre{g.logM[im], g.logN[jn], g.M[im], g.N[jn]};
}

__device__ __forceinline__ void produce_tile(const TablesDev& t, const GridDev& g,
                                             const GridLaunch& gl, int warp, int lane,
                                             const RowPre& rp, int slab, uint8_t* buf) {
  uint64_t* sD = reinterpret_cast<uint64_t*>(buf + gl.b_sD);
  int32_t* sP = reinterpret_cast<int32_t*>(buf + gl.b_sP);
  ClassRow* scls = reinterpret_cast<ClassRow*>(buf + gl.b_cls);
  if (warp == 0) {
    // member-class staircases: prefix minimum of D in member (scan) order
    const double qm = rp.qm, qn = rp.qn;
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
  } else if (gl.mode <= 1) {
    // tiles per (m, n) and the curve-major wave-scale table W[c][ib]
    uint64_t* T = reinterpret_cast<uint64_t*>(buf + gl.b_T);
    double* W = reinterpret_cast<double*>(buf + gl.b_W);
    const uint64_t m = rp.m, n = rp.n;
    const int ib0 = slab * gl.bper;
    const int nb = min(int(g.b_hi - g.b_lo), ib0 + gl.bper) - ib0;
    for (int wc = lane + 32 * (warp - 1); wc < t.NW; wc += 32 * (kProducerWarps - 1)) {
      const int c = t.wc_rep[wc];  // every curve of the class has these parameters
      const uint64_t tmn = ceil_div_c(t, c, 0, m, t.tile_m[c]) *
                           ceil_div_c(t, c, 1, n, t.tile_n[c]) * t.split_k[c];
      T[wc] = tmn;
      if (gl.mode == 0) {
        const uint64_t bpw = t.bpw[c];
        for (int ib = 0; ib < nb; ++ib)
          W[wc * nb + ib] =
              wave_scale(t, c, ceil_div_c(t, c, 2, g.B[g.b_lo + ib0 + ib] * tmn, bpw));
      }
    }
  }
}

template <bool VERIFY, int MODE, int NEAR, int NB>
__device__ __forceinline__ void consume_tile(const TablesDev& t, const GridDev& g,
                                             const GridLaunch& gl, const double* base_tab,
                                             const LaunchOut& out, int ctid, int row, int slab,
                                             int k_lo, int k_hi,
                                             const uint8_t* buf, const int2* gcur,
                                             const int32_t* gst, const double* glk) {
  const uint64_t* sD = reinterpret_cast<const uint64_t*>(buf + gl.b_sD);
  const int32_t* sP = reinterpret_cast<const int32_t*>(buf + gl.b_sP);
  const ClassRow* scls = reinterpret_cast<const ClassRow*>(buf + gl.b_cls);
  const uint64_t* T = reinterpret_cast<const uint64_t*>(buf + gl.b_T);
  const double* W = reinterpret_cast<const double*>(buf + gl.b_W);
  const RowView rv{scls, sD, sP};
  const int nN = int(g.nN), nK = int(g.nK);
  const int ib0 = slab * gl.bper;
  const int nb = min(int(g.b_hi - g.b_lo), ib0 + gl.bper) - ib0;
  uint64_t dmin1 = 0;
  int lastpos1 = 0;
  if (NEAR == 2) {
    dmin1 = scls[0].dmin;
    lastpos1 = scls[0].lastpos;
  }
  const int64_t plane = g.nM * g.nN * g.nK;
  double* const obase = out.lat + int64_t(ib0) * plane + int64_t(row) * nK;
  if (NEAR == 2 && MODE == 0 && !VERIFY && NB > 0) {
    // hot path, software-pipelined in groups of U k values: all kinfo loads,
    // then all nearest searches, then all base-table loads in flight
    // together, then the stores
    constexpr int U = 4;
    for (int k0 = k_lo; k0 < k_hi; k0 += U * kConsumers) {
      double2 ki[U];
      int ik[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        ik[u] = k0 + u * kConsumers + ctid;
        ki[u] = ik[u] < k_hi ? *reinterpret_cast<const double2*>(&g.kinfo[ik[u]])
                             : make_double2(0.0, 0.0);
      }
      int ci[U], wc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ik[u] < k_hi) {
          const int2 gp = nearest_one_class(t.G, glk, rv, dmin1, lastpos1, ki[u].x,
                                            __double2loint(ki[u].y));
          const int2 cw = gcur[gst[gp.x] + gp.y];
          ci[u] = cw.x;
          wc[u] = cw.y;
        } else {
          ci[u] = -2;  // beyond the k axis
          wc[u] = 0;
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
        const double* w = W + wc[u] * NB;
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) o[ib * plane] = __dmul_rn(bv[u], w[ib]);
      }
    }
    return;
  }
  const int im = row / nN, jn = row - im * nN;
  for (int ik = k_lo + ctid; ik < k_hi; ik += kConsumers) {
    const double2 ki = *reinterpret_cast<const double2*>(&g.kinfo[ik]);
    const int start = __double2loint(ki.y);
    int ci;
    if (NEAR == 2) {
      const int2 gp = nearest_one_class(t.G, glk, rv, dmin1, lastpos1, ki.x, start);
      ci = gcur[gst[gp.x] + gp.y].x;
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
    const int wci = t.wc_of[ci];
    if (MODE == 0 && !VERIFY) {
      const double* w = W + wci * nb;
      for (int ib = 0; ib < nb; ++ib, o += plane) *o = __dmul_rn(base, w[ib]);
      continue;
    }
    const uint64_t k = g.K[ik];
    // the curve's parameters once per k (registers), then the slab's batch
    // values in arithmetic only
    const WcParam cpar = MODE == 2 ? curve_params(t, ci) : WcParam{};
    const bool crb = MODE == 2 ? t.rowblock[ci] != 0 : false;
    const uint64_t m_val = MODE == 2 ? g.M[im] : 0, n_val = MODE == 2 ? g.N[jn] : 0;
    for (int ib = 0; ib < nb; ++ib, o += plane) {
      const uint64_t b = g.B[g.b_lo + ib0 + ib];
      double lat;
      uint64_t blocks, waves;
      if (MODE <= 1) {
        blocks = b * T[wci];
        waves = ceil_div_c(t, ci, 2, blocks, t.bpw[ci]);
        lat = __dmul_rn(base, wave_scale(t, ci, waves));
      } else {
        const PointResult r = predict_point_p(cpar, crb, b, m_val, n_val, k, base);
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

template <bool VERIFY, int MODE, int NEAR, int NB>
__global__ void __launch_bounds__(kWsThreads) grid_kernel(TablesDev t, GridDev g, GridLaunch gl,
                                                          const double* __restrict__ base_tab,
                                                          LaunchOut out) {
  extern __shared__ __align__(16) uint8_t smem[];
  int2* gcur = reinterpret_cast<int2*>(smem + gl.off_gcur);
  int32_t* gst = reinterpret_cast<int32_t*>(smem + gl.off_gst);
  double* glk = reinterpret_cast<double*>(smem + gl.off_glk);
  uint8_t* bufs = smem + gl.off_buf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // tile-independent candidate tables: (curve, wave class) per group position
  for (int j = tid; j < t.R; j += blockDim.x) {
    const int c = t.g_curve[j];
    gcur[j] = make_int2(c, c >= 0 ? t.wc_of[c] : -1);
  }
  for (int j = tid; j < t.G; j += blockDim.x) {
    gst[j] = t.grp_start[j];
    glk[j] = t.grp_lk[j];
  }
  __syncthreads();
  if (warp < kProducerWarps) {
    if (g.dev_planned) pdl_wait();  // row logs come from the planner kernel
    int it = 0;
    int tile = blockIdx.x;
    // tile = (row * nbs + slab) * nkt + k tile
    RowPre cur = tile < gl.tiles ? load_row(g, tile / gl.nkt / gl.nbs) : RowPre{};
    for (; tile < gl.tiles; tile += gridDim.x, ++it) {
      const int nt = tile + gridDim.x;
      const RowPre nxt = nt < gl.tiles ? load_row(g, nt / gl.nkt / gl.nbs) : cur;  // prefetch
      const int b = it & 1;
      if (it >= 2) named_sync(kBarEmpty + b, kWsThreads);
      produce_tile(t, g, gl, warp, lane, cur, (tile / gl.nkt) % gl.nbs, bufs + b * gl.buf_bytes);
      named_arrive(kBarFull + b, kWsThreads);
      cur = nxt;
    }
    // complete the consumers' last EMPTY arrivals (every barrier instance full)
    for (int j = max(0, it - 2); j < it; ++j) named_sync(kBarEmpty + (j & 1), kWsThreads);
  } else {
    pdl_wait();  // base table complete and visible
    const int ctid = tid - 32 * kProducerWarps;
    int it = 0;
    for (int tile = blockIdx.x; tile < gl.tiles; tile += gridDim.x, ++it) {
      const int b = it & 1;
      named_sync(kBarFull + b, kWsThreads);
      const int rs = tile / gl.nkt, kx = tile - rs * gl.nkt;
      const int k_lo = kx * gl.kt, k_hi = min(int(g.nK), k_lo + gl.kt);
      consume_tile<VERIFY, MODE, NEAR, NB>(t, g, gl, base_tab, out, ctid, rs / gl.nbs,
                                           rs % gl.nbs, k_lo, k_hi, bufs + b * gl.buf_bytes,
                                           gcur, gst, glk);
      named_arrive(kBarEmpty + b, kWsThreads);
    }
  }
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
  if (gl.tiles == 0) return cudaSuccess;
  // programmatic dependent launch: tile setup overlaps the base-table kernel;
  // griddepcontrol.wait guards the first base-table read
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(gl.ctas));
  cfg.blockDim = dim3(kWsThreads);
  cfg.dynamicSmemBytes = size_t(gl.smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, t, g, gl, base, out);
}

}  // namespace

cudaError_t launch_sweep(const TablesDev& t, const GridDev& g, const GridLaunch& gl,
                         const double* base, const LaunchOut& out, cudaStream_t s) {
  if (out.curve != nullptr)
    return gl.mode == 0 ? launch_grid_t<true, 0>(t, g, gl, base, out, s)
           : gl.mode == 1 ? launch_grid_t<true, 1>(t, g, gl, base, out, s)
                          : launch_grid_t<true, 2>(t, g, gl, base, out, s);
  return gl.mode == 0 ? launch_grid_t<false, 0>(t, g, gl, base, out, s)
         : gl.mode == 1 ? launch_grid_t<false, 1>(t, g, gl, base, out, s)
                        : launch_grid_t<false, 2>(t, g, gl, base, out, s);
}

}  // namespace gk
}  // namespace pm2l
