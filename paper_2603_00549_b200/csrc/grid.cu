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
#include <cstdio>
#include <cstdlib>

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

__global__ void __launch_bounds__(256) base_table_kernel(TablesDev t, GridDev g,
                                                         const uint64_t* __restrict__ K, int nK,
                                                         double* __restrict__ base,
                                                         double* __restrict__ fixval,
                                                         unsigned long long* stats) {
  pdl_release();  // the grid kernel may start its (independent) row setup now
  // the launch's unresolved-point statistics start here (the grid kernel
  // touches them only after griddepcontrol.wait)
  if (stats && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    stats[0] = ~0ull;
    stats[1] = 0ull;
    stats[2] = 0ull;
  }
  __shared__ double sd[kMaxSmemSamples], sy[kMaxSmemSamples];
  const int c = blockIdx.y;
  if (c == t.C) {  // exact-record hits: their final latency, applied after the grid kernel
    if (!fixval) return;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < g.n_fix;
         i += int64_t(gridDim.x) * blockDim.x) {
      const uint64_t* c4 = g.fix_coord + 4 * i;
      const int ci = g.fix_curve[i];
      fixval[i] = ci < 0 ? qnan()
                         : predict_point(t, ci, c4[0], c4[1], c4[2], c4[3], base_of(t, ci, c4[3])).lat;
    }
    return;
  }
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
// Warp-specialised, persistent: each CTA has kProducerWarps producer warps
// and kConsumerWarps consumer warps and walks (row, batch-slab) tiles with a
// stride of gridDim.x.  Producers build the next tile's row state into one of
// two shared-memory buffers while consumers compute the current tile's points
// from the other; the hand-off uses named barriers (FULL/EMPTY per buffer).
constexpr int kProducerWarps = 2;   // warp 0: staircases, warp 1: Tmn / W
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kWsThreads = 32 * (kProducerWarps + kConsumerWarps);

struct GridLaunch {
  int tiles;     // rows * nbs * nkt
  int nkt, kt;   // k tiles per (row, slab) and k values per k tile
  int kpt;       // k values per consumer thread
  int nbs;       // batch slabs
  int bper;      // batch values per slab
  int mode;      // 0: GEMM + W table, 1: GEMM per point, 2: general (row-block)
  int near;      // 0: general sweep, 1: sweep + tie mask (G <= 32), 2: one member class
  int ctas;      // persistent CTAs
  // shared memory: constant part, then two row-state buffers
  int off_gcur, off_gst, off_glk, off_buf, buf_bytes;
  int b_sD, b_sP, b_cls, b_T, b_W;  // offsets inside a buffer
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
  gl.off_gcur = take(8ll * t.R);
  gl.off_gst = take(4ll * t.G);
  gl.off_glk = take(8ll * t.G);
  gl.off_buf = int(o);
  int64_t bo = 0;
  auto btake = [&](int64_t bytes) {
    const int64_t at = bo;
    bo = (bo + bytes + 15) & ~int64_t(15);
    return int(at);
  };
  gl.b_sD = btake(8ll * t.CM);
  gl.b_sP = btake(4ll * t.CM);
  gl.b_cls = btake(16ll * t.NC);
  gl.b_T = btake(gl.mode <= 1 ? 8ll * t.NW : 0);
  gl.b_W = btake(gl.mode == 0 ? 8ll * t.NW * gl.bper : 0);
  gl.buf_bytes = int(bo);
  gl.smem = o + 2 * bo;
}

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

// ------------------------------------------------- one-class lookup path
// The one-class argmin (nearest_one_class) splits into a k-only part and a
// row-only part:
//   case A  (mn(k) <= dmin): group = leftmost group with dk(g, k) <= dmin,
//                            member = lastpos
//   case B  (mn(k) >  dmin): group = gB(k), member = staircase(mn(k))
// mn, gB and rank(k) (position of k in the descending order of mn inside its
// k chunk) are k-only and come from the host (GridDev::kfast / mn_sorted).
// Per (row, k chunk) one warp turns the row's staircase into cut points
//   cut[s]  = #{ranks with mn >= sD[s]}  (s < len-1);  cut[len-1] = #{mn > dmin}
//   kap[g]  = first k index at which group g lies left of log2 k AND is
//             farther than dmin from it (monotone in k: a binary search;
//             non-decreasing in g)
// and expands them into two byte maps over the chunk
//   rmap[rank] = staircase step of mn (case B) or 0xFF (case A)
//   gmap[ik]   = #{g : kap[g] <= ik} = the case-A group
// so resolving one k is three shared-memory lookups.  Every comparison is
// the one nearest_one_class makes, on the same bits: the argmin is identical.
//
// Warp-autonomous: each warp builds its tile's state and then writes the
// tile's points; many independent tiles are in flight per SM and no barrier
// couples warps.
constexpr int kRowWarps = 8;
constexpr int kRingProd = 4;   // grid_ring_kernel: default builder warps per CTA
constexpr int kRingSlots = 6;  // default tile-state slots per CTA
constexpr int kRingMaxSlots = 16;

#ifdef PM2L_TIMING
// diagnostic build only (tools/row_timing.py): per-tile phase timestamps
__device__ unsigned long long g_row_dbg[16384 * 8];
__device__ unsigned long long g_pdl_dbg[4096 * 4];  // per CTA: entry, before/after pdl wait, first FULL
#define ROW_MARK(tile, i)                                                         \
  do {                                                                            \
    if (lane == 0 && (tile) < 16384) {                                            \
      g_row_dbg[(tile) * 8 + (i)] = clock64();                                    \
    }                                                                             \
  } while (0)
#else
#define ROW_MARK(tile, i) do {} while (0)
#endif

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
// TMA bulk copy global -> shared (bytes: multiple of 16, both ends 16-aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__host__ __device__ constexpr uint32_t r16(int64_t b) { return uint32_t((b + 15) & ~int64_t(15)); }

// n / d for n < 2^31 through a host-computed u32 magic (Granlund-Montgomery)
struct FastDiv {
  uint32_t m, s;  // multiplier, sh1 | sh2 << 8
};
inline FastDiv fast_div_for(uint32_t d) {
  int l = 0;
  while ((uint64_t(1) << l) < d) ++l;
  const uint64_t m = ((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1;
  return FastDiv{uint32_t(m), uint32_t(l < 1 ? l : 1) | (uint32_t(l > 1 ? l - 1 : 0) << 8)};
}
__device__ __forceinline__ int fdiv(int n, FastDiv f) {
  const uint32_t q = __umulhi(f.m, uint32_t(n));
  return int((q + ((uint32_t(n) - q) >> (f.s & 0xFF))) >> (f.s >> 8));
}

struct RowLaunch {
  int tiles, nbs, nkc, kc;   // tiles = rows * nbs * nkc; k chunk length (even)
  FastDiv d_nkc, d_nbs, d_nN;
  int seg;                   // byte-map bytes per lane (multiple of 16)
  int ring;                  // producer/consumer variant (grid_ring_kernel)
  int pair;                  // 16-byte pair stores (even k axis, aligned output)
  int rowblock;              // row-block tables: per-point wave scale (ring kernel, pairs)
  int prod, slots;           // ring: builder warps, tile-state slots
  int ctas;
  int off_bar, off_gcur, off_glk, off_clm, off_cln, off_wcp, off_kf, off_ms, off_kq, off_kr, off_warp;
  int w_hdr, w_sD, w_sP, w_cut, w_W, w_rmap, w_gmap, warp_bytes;
  int64_t smem;
};

void row_layout(const TablesDev& t, const GridDev& g, int nb, bool stage_k, RowLaunch& rl) {
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = (o + bytes + 15) & ~int64_t(15);
    return int(at);
  };
  rl.off_bar = take(8ll * (2 + 4 * kRingMaxSlots));  // prologue + ring FULL/EMPTY/W-/stair-ready
  rl.off_gcur = take(8ll * t.R);
  rl.off_glk = take(8ll * t.G);
  rl.off_clm = take(8ll * t.CM);
  rl.off_cln = take(8ll * t.CM);
  rl.off_wcp = take(int64_t(sizeof(WcParam)) * t.NW);
  rl.seg = int(kmap_lane_bytes(g.nK));
  rl.off_kf = take(stage_k ? 4ll * g.nK : 0);
  rl.off_ms = take(stage_k ? 8ll * g.nK : 0);
  rl.off_kq = take(stage_k ? 8ll * g.nK : 0);
  rl.off_kr = take(stage_k ? 4ll * rl.nkc * t.G : 0);
  rl.off_warp = int(o);
  int64_t w = 0;
  auto wtake = [&](int64_t bytes) {
    const int64_t at = w;
    w = (w + bytes + 15) & ~int64_t(15);
    return int(at);
  };
  rl.w_hdr = wtake(16);
  rl.w_sD = wtake(8ll * t.CM);
  rl.w_sP = wtake(4ll * t.CM);
  rl.w_cut = wtake(4ll * (t.CM + t.G + 1));
  rl.w_W = wtake(8ll * t.NW * nb);
  rl.w_rmap = wtake(32ll * rl.seg);
  rl.w_gmap = wtake(32ll * rl.seg);
  rl.warp_bytes = int(w);
  rl.smem = o + int64_t(rl.ring ? rl.slots : kRowWarps) * w;
}

__device__ __forceinline__ uint64_t lds_u64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint64_t ceil_div_w(const WcParam& p, int j, uint64_t a, uint64_t d) {
  const uint64_t num = a + d - 1;
  const uint32_t s = p.ds[j];
  if ((s >> 16) && num <= 0xFFFFFFFFull) {
    const uint32_t n32 = uint32_t(num);
    const uint32_t q = __umulhi(p.dm[j], n32);
    return uint64_t((q + ((n32 - q) >> (s & 0xFF))) >> ((s >> 8) & 0xFF));
  }
  return udiv_slow(num, d);
}

// Row scalars of one tile (loaded one tile ahead).
template <int NB>
struct RowIn {
  double qm, qn;
  int im, jn;
  uint64_t b[NB];
  uint64_t cm[2], cn[2];  // tile counts of wave classes lane, lane + 32
};

template <int NB, bool RB = false>
__device__ __forceinline__ RowIn<NB> load_row_in(const GridDev& g, const RowLaunch& rl, int tile,
                                                 int NW, int lane) {
  RowIn<NB> r;
  const int rs = fdiv(tile, rl.d_nkc), row = fdiv(rs, rl.d_nbs), slab = rs - row * rl.nbs;
  const int im = fdiv(row, rl.d_nN), jn = row - im * int(g.nN);
  r.qm = g.logM[im];
  r.qn = g.logN[jn];
  r.im = im;
  r.jn = jn;
#pragma unroll
  for (int ib = 0; ib < NB; ++ib) r.b[ib] = g.B[g.b_lo + slab * NB + ib];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int wc = min(lane + 32 * h, NW - 1);
    r.cm[h] = RB ? 0 : g.cm_tab[im * NW + wc];   // row-block waves ignore (m, n)
    r.cn[h] = RB ? 0 : g.cn_tab[jn * NW + wc];
  }
  return r;
}

// Shared-memory views and table pointers common to the row kernels.
template <bool STAGE>
struct RowCtx {
  int2* gcur;
  double *glk, *clm, *cln;
  WcParam* wcp;
  const uint32_t* kfs;
  const uint64_t* ms;    // per-k tables (shared when STAGE)
  const double* kq;
  const int32_t* krt;    // [chunk x G] kright
  uint32_t ms_s, kq_s;   // shared addresses of ms / kq (STAGE)
  int G, CM, NW, nK;
  int64_t plane;
};

template <bool STAGE>
__device__ __forceinline__ RowCtx<STAGE> row_ctx(uint8_t* smem, const TablesDev& t, const GridDev& g,
                                                 const RowLaunch& rl) {
  RowCtx<STAGE> c;
  c.gcur = reinterpret_cast<int2*>(smem + rl.off_gcur);
  c.glk = reinterpret_cast<double*>(smem + rl.off_glk);
  c.clm = reinterpret_cast<double*>(smem + rl.off_clm);
  c.cln = reinterpret_cast<double*>(smem + rl.off_cln);
  c.wcp = reinterpret_cast<WcParam*>(smem + rl.off_wcp);
  c.kfs = STAGE ? reinterpret_cast<const uint32_t*>(smem + rl.off_kf) : g.kfast;
  c.ms = STAGE ? reinterpret_cast<const uint64_t*>(smem + rl.off_ms) : g.mn_sorted;
  c.kq = STAGE ? reinterpret_cast<const double*>(smem + rl.off_kq) : g.logK;
  c.krt = STAGE ? reinterpret_cast<const int32_t*>(smem + rl.off_kr) : g.kright;
  c.ms_s = smem_u32(smem + rl.off_ms);
  c.kq_s = smem_u32(smem + rl.off_kq);
  c.G = t.G; c.CM = t.CM; c.NW = t.NW; c.nK = int(g.nK);
  c.plane = g.nM * g.nN * g.nK;
  return c;
}

// Prologue (thread 0): CTA-constant tables by TMA bulk copies on two
// mbarriers, the small tables first (the staircase and W table need only
// those), the per-k tables behind them.
template <bool STAGE>
__device__ __forceinline__ void row_prologue(uint8_t* smem, const RowCtx<STAGE>& c, const TablesDev& t,
                                             const GridDev& g, const RowLaunch& rl, uint64_t* bar) {
  mbar_expect_tx(bar, r16(8ll * t.R) + r16(8ll * c.G) + 2 * r16(8ll * c.CM) +
                          r16(int64_t(sizeof(WcParam)) * c.NW));
  bulk_g2s(c.clm, t.cls_lm, r16(8ll * c.CM), bar);
  bulk_g2s(c.cln, t.cls_ln, r16(8ll * c.CM), bar);
  bulk_g2s(c.wcp, t.wcp, r16(int64_t(sizeof(WcParam)) * c.NW), bar);
  bulk_g2s(c.glk, t.grp_lk, r16(8ll * c.G), bar);
  bulk_g2s(c.gcur, t.g_cw, r16(8ll * t.R), bar);
  if (STAGE) {
    mbar_expect_tx(bar + 1, r16(4ll * c.nK) + 2 * r16(8ll * c.nK) + r16(4ll * rl.nkc * c.G));
    bulk_g2s(smem + rl.off_ms, g.mn_sorted, r16(8ll * c.nK), bar + 1);
    bulk_g2s(smem + rl.off_kq, g.logK, r16(8ll * c.nK), bar + 1);
    bulk_g2s(smem + rl.off_kr, g.kright, r16(4ll * rl.nkc * c.G), bar + 1);
    bulk_g2s(smem + rl.off_kf, g.kfast, r16(4ll * c.nK), bar + 1);
  }
}

// Tile coordinates: tile = (row * nbs + slab) * nkc + k chunk.
struct TileXY {
  int row, slab, kcx, k0, kc;
};
__device__ __forceinline__ TileXY tile_xy(const RowLaunch& rl, int tile, int nK) {
  TileXY x;
  const int rs = fdiv(tile, rl.d_nkc);
  x.kcx = tile - rs * rl.nkc;
  x.row = fdiv(rs, rl.d_nbs);
  x.slab = rs - x.row * rl.nbs;
  x.k0 = x.kcx * rl.kc;
  x.kc = min(rl.kc, nK - x.k0);
  return x;
}

// Wave-scale table W[wave class][ib] of one tile's (m, n) and batch slab.
template <int NB, bool STAGE>
__device__ __forceinline__ void build_w_table(const RowCtx<STAGE>& c, const GridDev& g,
                                              const RowIn<NB>& cur, double* W, int lane) {
  const int NW = c.NW;
  for (int wc = lane; wc < NW; wc += 32) {
    const WcParam& p = c.wcp[wc];
    const uint64_t tmn = wc < 64 ? cur.cm[wc >> 5] * cur.cn[wc >> 5]
                                 : g.cm_tab[cur.im * NW + wc] * g.cn_tab[cur.jn * NW + wc];
    const double rw = p.rw;
#pragma unroll
    for (int ib = 0; ib < NB; ++ib) {
      const double w = __ull2double_rn(ceil_div_w(p, 2, cur.b[ib] * tmn, p.bpw));
      W[wc * NB + ib] = rw == 1.0 ? w : __ddiv_rn(w, rw);
    }
  }
}

// One tile's lookup state (one warp): staircase, wave-scale table, cut
// points, byte maps, written into the slot `wb`; len / lastpos into its
// header.
template <int NB, bool STAGE, int SEGW, bool RB = false>
__device__ __forceinline__ void build_tile(const RowCtx<STAGE>& c, const GridDev& g,
                                           const RowLaunch& rl, const TileXY& x,
                                           const RowIn<NB>& cur, uint8_t* wb, int lane,
                                           int mark_tile = 1 << 30, bool with_w = true,
                                           uint64_t* stair_ready = nullptr) {
  // stair_ready != nullptr: a helper warp builds the group cuts and gmap of
  // this tile (help_group_map) once the staircase is published
  uint64_t* sD = reinterpret_cast<uint64_t*>(wb + rl.w_sD);
  int32_t* sP = reinterpret_cast<int32_t*>(wb + rl.w_sP);
  double* W = reinterpret_cast<double*>(wb + rl.w_W);
  int32_t* hdr = reinterpret_cast<int32_t*>(wb + rl.w_hdr);
  const int CM = c.CM, NW = c.NW;
  // ---- staircase: prefix minimum of D_j = max(|lm_j-qm|, |ln_j-qn|)
  uint64_t dmin = ~0ull;
  int len = 0, lastpos = 0;
  auto dist = [&](int j) {
    return umax64(abs_bits(__dsub_rn(c.clm[j], cur.qm)), abs_bits(__dsub_rn(c.cln[j], cur.qn)));
  };
  if (CM <= 64) {
    // one warp scan: members 2*lane, 2*lane + 1 per lane
    const int ja = 2 * lane, jb = ja + 1;
    const uint64_t da = ja < CM ? dist(ja) : ~0ull, db = jb < CM ? dist(jb) : ~0ull;
    uint64_t pm = umin64(da, db);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, pm, off);
      if (lane >= off && o < pm) pm = o;
    }
    uint64_t excl = __shfl_up_sync(0xFFFFFFFFu, pm, 1);
    if (lane == 0) excl = ~0ull;
    const bool ra = ja < CM && da < excl;
    const bool rb = jb < CM && db < umin64(excl, da);
    const unsigned ma = __ballot_sync(0xFFFFFFFFu, ra), mb = __ballot_sync(0xFFFFFFFFu, rb);
    const unsigned below = (1u << lane) - 1u;
    const int pa = __popc(ma & below) + __popc(mb & below);
    if (ra) { sD[pa] = da; sP[pa] = ja; }
    if (rb) { sD[pa + ra] = db; sP[pa + ra] = jb; }
    len = __popc(ma) + __popc(mb);
    const int hi = 31 - __clz(ma | mb);  // ma | mb != 0: member 0 is a record
    lastpos = ((mb >> hi) & 1u) ? 2 * hi + 1 : 2 * hi;
    dmin = __shfl_sync(0xFFFFFFFFu, pm, 31);
  } else for (int b0 = 0; b0 < CM; b0 += 32) {
    const int j = b0 + lane;
    const uint64_t d = j < CM ? dist(j) : ~0ull;
    uint64_t pm = d;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint64_t o = __shfl_up_sync(0xFFFFFFFFu, pm, off);
      if (lane >= off && o < pm) pm = o;
    }
    uint64_t excl = __shfl_up_sync(0xFFFFFFFFu, pm, 1);
    if (lane == 0) excl = ~0ull;
    if (dmin < excl) excl = dmin;
    const bool rec = j < CM && d < excl;
    const unsigned mask = __ballot_sync(0xFFFFFFFFu, rec);
    if (rec) {
      const int pos = len + __popc(mask & ((1u << lane) - 1u));
      sD[pos] = d;
      sP[pos] = j;
    }
    if (mask) lastpos = b0 + 31 - __clz(mask);
    len += __popc(mask);
    const uint64_t tail = __shfl_sync(0xFFFFFFFFu, pm, 31);
    if (tail < dmin) dmin = tail;
  }
  ROW_MARK(mark_tile, 5);
  const bool with_g = stair_ready == nullptr;
  if (!with_g) {  // publish len and dmin for the helper
    if (lane == 0) {
      hdr[0] = len;
      *reinterpret_cast<uint64_t*>(hdr + 2) = dmin;
    }
    __syncwarp();
    mbar_arrive(stair_ready);
  }
  // ---- wave-scale table W[wave class][ib] of this (m, n) and batch slab
  if (with_w && !RB) build_w_table<NB, STAGE>(c, g, cur, W, lane);
  if (RB) {  // row-block waves depend on (b, k): the writers need the slab's batch values
#pragma unroll
    for (int ib = 0; ib < NB; ++ib)
      if (lane == ib) W[ib] = __longlong_as_double(static_cast<long long>(cur.b[ib]));
  }
  __syncwarp();
  ROW_MARK(mark_tile, 6);
  // ---- cut points: fixed-trip branch-free binary searches, one shared
  // load per step, both kinds in one loop (lanes never diverge)
  //   i < len : #{ranks r: mn(r) >= sD[i]} (i == len-1: > dmin); mn descends
  //   i >= len: #{k: NOT (group i-len left of log2 k and farther than dmin)}
  //             = kright + #{k >= kright: log2 k - lk <= dmin}
  constexpr int SL = SEGW * 4;
  int32_t* cut = reinterpret_cast<int32_t*>(wb + rl.w_cut);
  {
    const int k0 = x.k0, kc = x.kc;
    int top = 1;
    while (top * 2 <= kc) top *= 2;
    for (int i = lane; i < len + (with_g ? c.G : 0); i += 32) {
      const bool rk = i < len, strict = i == len - 1;
      const int gg = rk ? 0 : i - len;
      const uint64_t xv = rk ? sD[i] : dmin;
      const double lk = c.glk[gg];
      const int kr = rk ? 0 : c.krt[x.kcx * c.G + gg];
      int lo = 0;
      for (int step = top; step; step >>= 1) {
        const int r = k0 + min(lo + step, kc) - 1;
        uint64_t v;
        if (STAGE) v = lds_u64((rk ? c.ms_s : c.kq_s) + 8u * uint32_t(r));
        else v = rk ? c.ms[r] : __double_as_longlong(c.kq[r]);
        const bool keep = rk ? (v > xv || (!strict && v == xv))
                             : (r - k0 < kr || abs_bits(__dsub_rn(__longlong_as_double(v), lk)) <= xv);
        lo += (lo + step <= kc && keep) ? step : 0;
      }
      cut[i] = lo;
    }
  }
  __syncwarp();
  ROW_MARK(mark_tile, 7);
  // ---- byte maps: map[r] = #{cuts <= r} (+ 0xFF from cut[len-1] on for
  // the rank map), one lane per SL consecutive bytes: a broadcast count of
  // the cuts before the segment, then SIMD increments for the few inside
  {
    constexpr int QW = SL / 8;  // u64 words per lane
    constexpr uint64_t kOnes = 0x0101010101010101ull;
    const int r0 = lane * SL;
    const int nr = len - 1, ng = with_g ? c.G : 0, ff = cut[len - 1];
    // first s with cut[s] > r0 in each cut list, both searches interleaved
    int b0 = 0, h0 = nr, b1 = 0, h1 = ng;
    const int32_t* cg = cut + len;
    while (b0 < h0 || b1 < h1) {
      const int m0 = (b0 + h0) >> 1, m1 = (b1 + h1) >> 1;
      const bool a0 = b0 < h0, a1 = b1 < h1;
      const int c0 = a0 ? cut[m0] : 0, c1 = a1 ? cg[m1] : 0;
      if (a0) { if (c0 <= r0) b0 = m0 + 1; else h0 = m0; }
      if (a1) { if (c1 <= r0) b1 = m1 + 1; else h1 = m1; }
    }
    uint64_t w0[QW], w1[QW];
#pragma unroll
    for (int q = 0; q < QW; ++q) {
      w0[q] = uint64_t(b0) * kOnes;
      w1[q] = uint64_t(b1) * kOnes;
    }
    auto bump = [&](uint64_t* w, int e) {
#pragma unroll
      for (int q = 0; q < QW; ++q) {
        const int sh = e - 8 * q;  // bytes >= sh of word q count this cut
        w[q] += sh <= 0 ? kOnes : sh >= 8 ? 0ull : (kOnes << (8 * sh));
      }
    };
    for (int s = b0; s < nr; ++s) {
      const int e = cut[s] - r0;
      if (e >= SL) break;
      bump(w0, e);
    }
    for (int s = b1; s < ng; ++s) {
      const int e = cut[len + s] - r0;
      if (e >= SL) break;
      bump(w1, e);
    }
#pragma unroll
    for (int q = 0; q < QW; ++q) {
      const int sh = ff - r0 - 8 * q;
      w0[q] |= sh <= 0 ? ~0ull : sh >= 8 ? 0ull : (~0ull << (8 * sh));
    }
    uint64_t* mw0 = reinterpret_cast<uint64_t*>(wb + rl.w_rmap) + lane * QW;
    uint64_t* mw1 = reinterpret_cast<uint64_t*>(wb + rl.w_gmap) + lane * QW;
#pragma unroll
    for (int q = 0; q < QW; q += 2) {
      *reinterpret_cast<ulonglong2*>(mw0 + q) = make_ulonglong2(w0[q], w0[q + 1]);
      if (with_g) *reinterpret_cast<ulonglong2*>(mw1 + q) = make_ulonglong2(w1[q], w1[q + 1]);
    }
  }
  if (lane == 0) {
    hdr[0] = len;
    hdr[1] = lastpos;
  }
}

// Helper warp's share of a tile build (first tiles of the ring kernel): the
// group cuts and gmap, from the staircase the builder published (len, dmin
// in the slot header).  Same searches and map construction as build_tile.
template <bool STAGE, int SEGW>
__device__ __forceinline__ void help_group_map(const RowCtx<STAGE>& c, const GridDev& g,
                                               const RowLaunch& rl, const TileXY& x, uint8_t* wb,
                                               int lane) {
  constexpr int SL = SEGW * 4;
  const int32_t* hdr = reinterpret_cast<const int32_t*>(wb + rl.w_hdr);
  const int len = hdr[0];
  const uint64_t dmin = *reinterpret_cast<const uint64_t*>(hdr + 2);
  int32_t* cg = reinterpret_cast<int32_t*>(wb + rl.w_cut) + len;
  const int k0 = x.k0, kc = x.kc, G = c.G;
  int top = 1;
  while (top * 2 <= kc) top *= 2;
  for (int gg = lane; gg < G; gg += 32) {
    const double lk = c.glk[gg];
    const int kr = c.krt[x.kcx * G + gg];
    int lo = 0;
    for (int step = top; step; step >>= 1) {
      const int r = k0 + min(lo + step, kc) - 1;
      const double q = STAGE ? __longlong_as_double(static_cast<long long>(lds_u64(c.kq_s + 8u * uint32_t(r))))
                             : c.kq[r];
      const bool keep = r - k0 < kr || abs_bits(__dsub_rn(q, lk)) <= dmin;
      lo += (lo + step <= kc && keep) ? step : 0;
    }
    cg[gg] = lo;
  }
  __syncwarp();
  constexpr int QW = SL / 8;
  constexpr uint64_t kOnes = 0x0101010101010101ull;
  const int r0 = lane * SL;
  int b = 0, h = G;
  while (b < h) {
    const int m = (b + h) >> 1;
    if (cg[m] <= r0) b = m + 1; else h = m;
  }
  uint64_t w[QW];
#pragma unroll
  for (int q = 0; q < QW; ++q) w[q] = uint64_t(b) * kOnes;
  for (int s2 = b; s2 < G; ++s2) {
    const int e = cg[s2] - r0;
    if (e >= SL) break;
#pragma unroll
    for (int q = 0; q < QW; ++q) {
      const int sh = e - 8 * q;
      w[q] += sh <= 0 ? kOnes : sh >= 8 ? 0ull : (kOnes << (8 * sh));
    }
  }
  uint64_t* mw = reinterpret_cast<uint64_t*>(wb + rl.w_gmap) + lane * QW;
#pragma unroll
  for (int q = 0; q < QW; q += 2)
    *reinterpret_cast<ulonglong2*>(mw + q) = make_ulonglong2(w[q], w[q + 1]);
}

// Row-block wave scale (compute.py:78-106, _kernels.pyx:123-132):
// blocks = ceil(b*k / tile_m), waves = ceil(blocks / blocks_per_wave),
// scale = waves / ref_waves -- from the wave class's staged parameters.
__device__ __forceinline__ double rb_scale(const WcParam& p, uint64_t b, uint64_t k) {
  // slot 1 of a row-block class = tile_m * blocks_per_wave (tables.cpp):
  // ceil(ceil(x / tm) / bpw) == ceil(x / (tm * bpw)) for integers, so one
  // magic division when x + tm*bpw - 1 fits 32 bits; else the two steps
  const uint64_t x = b * k, num = x + p.tn - 1;
  uint64_t waves;
  if ((p.ds[1] >> 16) && num <= 0xFFFFFFFFull) {
    const uint32_t n32 = uint32_t(num), s = p.ds[1];
    const uint32_t q = __umulhi(p.dm[1], n32);
    waves = (q + ((n32 - q) >> (s & 0xFF))) >> ((s >> 8) & 0xFF);
  } else {
    waves = ceil_div_w(p, 2, ceil_div_w(p, 0, x, p.tm), p.bpw);
  }
  const double w = __ull2double_rn(waves);
  return p.rw == 1.0 ? w : __ddiv_rn(w, p.rw);
}

// Write one tile's points from its slot: 32-pair blocks b0, b0 + bstep, ...
// (two adjacent k per lane, one 16-byte store per batch value), then the
// exact-record hits that fall in those blocks.
template <int NB, bool STAGE, bool PAIR, bool RB = false>
__device__ __forceinline__ void emit_tile(const RowCtx<STAGE>& c, const TablesDev& t,
                                          const GridDev& g, const RowLaunch& rl, const TileXY& x,
                                          const uint8_t* wb, const double* __restrict__ base_tab,
                                          const LaunchOut& out, int b0, int bstep, int lane) {
  const int32_t* sP = reinterpret_cast<const int32_t*>(wb + rl.w_sP);
  const double* W = reinterpret_cast<const double*>(wb + rl.w_W);
  const uint8_t* rmap = wb + rl.w_rmap;
  const uint8_t* gmap = wb + rl.w_gmap;
  const int32_t* hdr = reinterpret_cast<const int32_t*>(wb + rl.w_hdr);
  const int lastpos = hdr[1], CM = c.CM, nK = c.nK, k0 = x.k0;
  const int64_t plane = c.plane;
  double* const obase = out.lat + int64_t(x.slab * NB) * plane + int64_t(x.row) * nK + k0;
  const double* const bbase = base_tab + k0;
  // pairs of adjacent k per lane; an odd chunk's last pair has no second k.
  // rl.pair: 16-byte pair stores (even k axis, 16-byte aligned output),
  // else two 8-byte stores
  const int nP = (x.kc + 1) >> 1, nB = (nP + 31) >> 5;
  constexpr bool pair = PAIR;
  auto has_second = [&](int p) { return PAIR || 2 * p + 1 < x.kc; };  // PAIR: kc even
  auto lookup = [&](uint32_t kf, int ikl) -> int2 {
    const uint32_t sb = rmap[kf & 0xFFFFu];
    const bool a = sb == 0xFFu;
    const int gg = a ? int(gmap[ikl]) : int((kf >> 16) & 0xFFu);
    const int pos = a ? lastpos : sP[sb];
    return c.gcur[gg * CM + pos];  // one class: group g's members at g * CM
  };
  constexpr int U = 4;
  for (int bq = b0; bq < nB; bq += U * bstep) {  // warp-uniform trip count (__all_sync)
    int2 v[U][2];
    int pp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      pp[u] = (bq + u * bstep) * 32 + lane;
      const int p = min(pp[u], nP - 1);
      const uint2 kf = *reinterpret_cast<const uint2*>(c.kfs + k0 + 2 * p);
      v[u][0] = lookup(kf.x, 2 * p);
      v[u][1] = has_second(p) ? lookup(kf.y, 2 * p + 1) : v[u][0];
    }
    bool all_ok = true;
#pragma unroll
    for (int u = 0; u < U; ++u) all_ok = all_ok && v[u][0].x >= 0 && v[u][1].x >= 0;
    if (RB) {
      // row-block families: per point scale from (b, k) and the wave class
      uint64_t bvals[NB];
#pragma unroll
      for (int ib = 0; ib < NB; ++ib)
        bvals[ib] = static_cast<uint64_t>(__double_as_longlong(W[ib]));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = pp[u];
        if (p >= nP) continue;
        double* o = obase + 2 * p;
        const bool has1 = has_second(p);
        const bool ok0 = v[u][0].x >= 0, ok1 = !has1 || v[u][1].x >= 0;
        const double bb0 = ok0 ? bbase[v[u][0].x * nK + 2 * p] : 0.0;
        const double bb1 = ok1 && has1 ? bbase[v[u][1].x * nK + 2 * p + 1] : 0.0;
        if (!(ok0 && ok1) && out.nan_stats) {
          atomicMin(out.nan_stats, (unsigned long long)(o - out.lat + (ok0 ? 1 : 0)));
          atomicAdd(out.nan_stats + 1, (unsigned long long)(NB * (2 - ok0 - ok1)));
        }
        const uint64_t ka = g.K[k0 + 2 * p], kb = has1 ? g.K[k0 + 2 * p + 1] : ka;
        const WcParam q0 = c.wcp[ok0 ? v[u][0].y : 0];
        const WcParam q1 = c.wcp[ok1 && has1 ? v[u][1].y : 0];
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) {
          const double a = ok0 ? __dmul_rn(bb0, rb_scale(q0, bvals[ib], ka)) : qnan();
          const double b = ok1 ? __dmul_rn(bb1, rb_scale(q1, bvals[ib], kb)) : qnan();
          if (PAIR) {
            *reinterpret_cast<double2*>(o + ib * plane) = make_double2(a, b);
          } else {
            o[ib * plane] = a;
            if (has1) o[ib * plane + 1] = b;
          }
        }
      }
    } else if (__all_sync(0xFFFFFFFFu, all_ok)) {
      double bv[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = min(pp[u], nP - 1);
        bv[u][0] = bbase[v[u][0].x * nK + 2 * p];
        bv[u][1] = has_second(p) ? bbase[v[u][1].x * nK + 2 * p + 1] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = pp[u];
        if (p >= nP) continue;
        double* o = obase + 2 * p;
        const double* w0 = W + v[u][0].y * NB;
        const double* w1 = W + v[u][1].y * NB;
#pragma unroll
        for (int ib = 0; ib < NB; ib += (NB >= 2 ? 2 : 1)) {
          double a0, a1, b0v, b1v;
          if (NB >= 2) {
            const double2 xw = *reinterpret_cast<const double2*>(w0 + ib);
            const double2 yw = *reinterpret_cast<const double2*>(w1 + ib);
            a0 = xw.x; a1 = xw.y; b0v = yw.x; b1v = yw.y;
          } else {
            a0 = w0[ib]; b0v = w1[ib]; a1 = b1v = 0.0;
          }
          const double r00 = __dmul_rn(bv[u][0], a0), r01 = __dmul_rn(bv[u][1], b0v);
          const double r10 = __dmul_rn(bv[u][0], a1), r11 = __dmul_rn(bv[u][1], b1v);
          if (pair) {
            *reinterpret_cast<double2*>(o + ib * plane) = make_double2(r00, r01);
            if (NB >= 2) *reinterpret_cast<double2*>(o + (ib + 1) * plane) = make_double2(r10, r11);
          } else {
            const bool has1 = has_second(p);
            o[ib * plane] = r00;
            if (has1) o[ib * plane + 1] = r01;
            if (NB >= 2) {
              o[(ib + 1) * plane] = r10;
              if (has1) o[(ib + 1) * plane + 1] = r11;
            }
          }
        }
      }
    } else {
      // some k resolves to a record without a curve: NaN + statistics
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int p = pp[u];
        if (p >= nP) continue;
        double* o = obase + 2 * p;
        const bool has1 = has_second(p);
        const bool ok0 = v[u][0].x >= 0, ok1 = !has1 || v[u][1].x >= 0;
        const double bb0 = ok0 ? bbase[v[u][0].x * nK + 2 * p] : 0.0;
        const double bb1 = ok1 && has1 ? bbase[v[u][1].x * nK + 2 * p + 1] : 0.0;
        if (!(ok0 && ok1) && out.nan_stats) {
          atomicMin(out.nan_stats, (unsigned long long)(o - out.lat + (ok0 ? 1 : 0)));
          atomicAdd(out.nan_stats + 1, (unsigned long long)(NB * (2 - ok0 - ok1)));
        }
        const double* w0 = W + (ok0 ? v[u][0].y : 0) * NB;
        const double* w1 = W + (ok1 && has1 ? v[u][1].y : 0) * NB;
#pragma unroll
        for (int ib = 0; ib < NB; ++ib) {
          const double a = ok0 ? __dmul_rn(bb0, w0[ib]) : qnan();
          const double b = ok1 ? __dmul_rn(bb1, w1[ib]) : qnan();
          if (pair) {
            *reinterpret_cast<double2*>(o + ib * plane) = make_double2(a, b);
          } else {
            o[ib * plane] = a;
            if (has1) o[ib * plane + 1] = b;
          }
        }
      }
    }
  }
  // exact-record hits in these blocks take priority over the nearest result
  // (_kernels.pyx:107-110): re-count them by their exact result
  const int f0 = g.fixr_off[x.row], f1 = g.fixr_off[x.row + 1];
  if (f1 > f0) {
    __syncwarp();  // this warp's stores above are visible to every lane
    for (int f = f0 + lane; f < f1; f += 32) {
      const FixEntry fe = g.fixr[f];
      const int ikl = fe.ik - k0;
      if (ikl < 0 || ikl >= x.kc || fe.ib < x.slab * NB || fe.ib >= x.slab * NB + NB) continue;
      if (((ikl >> 6) - b0) % bstep != 0 || (ikl >> 6) < b0) continue;  // another warp's block
      double* o = out.lat + int64_t(fe.ib) * plane + int64_t(x.row) * nK + fe.ik;
      const int ci = fe.curve;
      if (out.nan_stats) {
        const bool was_nan = *o != *o;
        if (was_nan && ci >= 0) {
          atomicAdd(out.nan_stats + 1, ~0ull);
          atomicOr(out.nan_stats + 2, 1ull);
        }
        if (!was_nan && ci < 0) {
          atomicAdd(out.nan_stats + 1, 1ull);
          atomicMin(out.nan_stats, (unsigned long long)(o - out.lat));
        }
      }
      if (ci < 0) {
        *o = qnan();
      } else {
        const uint64_t* c4 = g.fix_coord + 4 * int64_t(fe.fix);
        *o = predict_point(t, ci, c4[0], c4[1], c4[2], c4[3], base_tab[ci * nK + fe.ik]).lat;
      }
    }
  }
}

// Warp-autonomous variant: each warp builds and writes its own tiles.
template <int NB, bool STAGE, int SEGW, bool PAIR>
__global__ void __launch_bounds__(32 * kRowWarps, 3) grid_row_kernel(TablesDev t, GridDev g,
                                                                    RowLaunch rl,
                                                                    const double* __restrict__ base_tab,
                                                                    LaunchOut out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + rl.off_bar);  // [0] tables, [1] per-k
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  ROW_MARK(blockIdx.x * kRowWarps + warp, 0);
  const RowCtx<STAGE> c = row_ctx<STAGE>(smem, t, g, rl);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    row_prologue<STAGE>(smem, c, t, g, rl, bar);
  }
  int tile = blockIdx.x * kRowWarps + warp;
  RowIn<NB> rin = load_row_in<NB>(g, rl, min(tile, rl.tiles - 1), t.NW, lane);  // in flight during the wait
  __syncthreads();  // mbarriers initialised before anyone waits on them
  mbar_wait(bar, 0);
  uint8_t* wb = smem + rl.off_warp + warp * rl.warp_bytes;
  bool waited = false, staged = !STAGE;
  for (; tile < rl.tiles; tile += gridDim.x * kRowWarps) {
    const TileXY x = tile_xy(rl, tile, c.nK);
    const RowIn<NB> cur = rin;
    {
      const int nt = tile + gridDim.x * kRowWarps;
      if (nt < rl.tiles) rin = load_row_in<NB>(g, rl, nt, t.NW, lane);  // next tile's scalars
    }
    ROW_MARK(tile, 1);
    if (!staged) {
      mbar_wait(bar + 1, 0);
      staged = true;
    }
    build_tile<NB, STAGE, SEGW>(c, g, rl, x, cur, wb, lane);
    __syncwarp();
    ROW_MARK(tile, 5);
    if (!waited) {
      pdl_wait();  // base table complete and visible
      waited = true;
    }
    ROW_MARK(tile, 6);
    emit_tile<NB, STAGE, PAIR>(c, t, g, rl, x, wb, base_tab, out, 0, 1, lane);
    __syncwarp();  // the warp's state buffers are rewritten by the next tile
    ROW_MARK(tile, 7);
  }
  if (!staged) mbar_wait(bar + 1, 0);  // never exit with bulk copies in flight
  if (!waited) pdl_wait();
}

// Producer/consumer variant: kRingProd builder warps fill kRingSlots
// shared-memory slots (mbarrier FULL/EMPTY per slot) with tile states, in
// the CTA's tile order; the other warps write the points, each taking every
// (kRowWarps - kRingProd)-th 32-pair block of a tile.  Writing starts after
// one tile's build and later builds proceed under the store stream.

template <int NB, bool STAGE, int SEGW, bool PAIR, bool RB>
__global__ void __launch_bounds__(32 * kRowWarps, 3) grid_ring_kernel(TablesDev t, GridDev g,
                                                                     RowLaunch rl,
                                                                     const double* __restrict__ base_tab,
                                                                     LaunchOut out) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + rl.off_bar);  // [0] tables, [1] per-k
  const int P = rl.prod, S = rl.slots, NC = kRowWarps - P;
  uint64_t* full = bar + 2;
  uint64_t* empty = full + S;
  // first P positions: writer warp w computes the W table of builder w's
  // first tile while that builder runs its staircase and searches
  uint64_t* wready = empty + S;
  uint64_t* sready = wready + kRingMaxSlots;  // builder's staircase published (first tiles)
  const int nhelp = min(P, min(NC, S));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const RowCtx<STAGE> c = row_ctx<STAGE>(smem, t, g, rl);
#ifdef PM2L_TIMING
  const unsigned long long t_entry = clock64();
#endif
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 32);
      mbar_init(empty + s, 32 * NC);
    }
    for (int s = 0; s < nhelp; ++s) {
      mbar_init(wready + s, 32);
      mbar_init(sready + s, 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    row_prologue<STAGE>(smem, c, t, g, rl, bar);
  }
  __syncthreads();  // mbarriers initialised before anyone waits on them
  if (warp < P) {
    int j = warp;
    int tile = blockIdx.x + j * gridDim.x;
    RowIn<NB> rin = load_row_in<NB, RB>(g, rl, min(tile, rl.tiles - 1), t.NW, lane);
    mbar_wait(bar, 0);
    if (STAGE) mbar_wait(bar + 1, 0);
    for (; tile < rl.tiles; j += P, tile += P * gridDim.x) {
      const int slot = j % S, use = j / S;
      const RowIn<NB> cur = rin;
      {
        const int nt = tile + P * gridDim.x;
        if (nt < rl.tiles) rin = load_row_in<NB, RB>(g, rl, nt, t.NW, lane);
      }
      if (use > 0) mbar_wait(empty + slot, (use - 1) & 1);
#ifdef PM2L_TIMING
      if (lane == 0 && tile < 16384) g_row_dbg[tile * 8] = t_entry;
#endif
      ROW_MARK(tile, 1);
      build_tile<NB, STAGE, SEGW, RB>(c, g, rl, tile_xy(rl, tile, c.nK), cur,
                                  smem + rl.off_warp + slot * rl.warp_bytes, lane, tile,
                                  /*with_w=*/j >= nhelp, j < nhelp ? sready + j : nullptr);
      __syncwarp();
      ROW_MARK(tile, 2);
      mbar_arrive(full + slot);
    }
  } else {
    const int cw = warp - P;
    if (cw < nhelp) {
      // W table of builder cw's first tile (position cw, slot cw)
      const int tile0 = blockIdx.x + cw * gridDim.x;
      if (tile0 < rl.tiles) {
        uint8_t* wb0 = smem + rl.off_warp + cw * rl.warp_bytes;
        const RowIn<NB> r0 = load_row_in<NB, RB>(g, rl, tile0, t.NW, lane);
        mbar_wait(bar, 0);
        if (!RB) build_w_table<NB, STAGE>(c, g, r0, reinterpret_cast<double*>(wb0 + rl.w_W), lane);
        if (STAGE) mbar_wait(bar + 1, 0);
        mbar_wait(sready + cw, 0);  // the builder's staircase is published
        help_group_map<STAGE, SEGW>(c, g, rl, tile_xy(rl, tile0, c.nK), wb0, lane);
      }
      __syncwarp();
      mbar_arrive(wready + cw);
    }
    mbar_wait(bar, 0);
    if (STAGE) mbar_wait(bar + 1, 0);
#ifdef PM2L_TIMING
    if (cw == 0 && lane == 0 && blockIdx.x < 4096) {
      g_pdl_dbg[blockIdx.x * 4] = t_entry;
      g_pdl_dbg[blockIdx.x * 4 + 1] = clock64();
    }
#endif
    pdl_wait();  // base table complete and visible
#ifdef PM2L_TIMING
    if (cw == 0 && lane == 0 && blockIdx.x < 4096) g_pdl_dbg[blockIdx.x * 4 + 2] = clock64();
#endif
    for (int j = 0, tile = blockIdx.x; tile < rl.tiles; ++j, tile += gridDim.x) {
      const int slot = j % S, use = j / S;
      mbar_wait(full + slot, use & 1);
      if (j < nhelp) mbar_wait(wready + j, 0);
#ifdef PM2L_TIMING
      if (j == 0 && cw == 0 && lane == 0 && blockIdx.x < 4096) g_pdl_dbg[blockIdx.x * 4 + 3] = clock64();
#endif
      if (cw == 0) ROW_MARK(tile, 3);
      emit_tile<NB, STAGE, PAIR, RB>(c, t, g, rl, tile_xy(rl, tile, c.nK),
                           smem + rl.off_warp + slot * rl.warp_bytes, base_tab, out, cw, NC,
                           lane);
      __syncwarp();
      if (cw == 0) ROW_MARK(tile, 4);
      mbar_arrive(empty + slot);
    }
  }
}

// Exact-record hits take priority over the nearest result (_kernels.pyx:107-110).
// `fixval` (nullable) holds their latencies, precomputed by the base-table
// kernel off the critical path.
template <bool VERIFY>
__global__ void fixup_kernel(TablesDev t, GridDev g, LaunchOut out, const double* fixval) {
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
  if (!VERIFY && fixval) {
    out.lat[p] = fixval[i];
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
  if (all_curves) {  // all_curves_kernel: (row, k tile, slab) CTAs of kThreads
    const int64_t target = 148 * 8;
    auto ktiles_for = [&](int kpt) {
      return int((g.nK + int64_t(kpt) * kThreads - 1) / (int64_t(kpt) * kThreads));
    };
    gl.kpt = 4;
    int ktiles = ktiles_for(gl.kpt);
    while (gl.kpt > 1 && rows * ktiles < target) {
      gl.kpt >>= 1;
      ktiles = ktiles_for(gl.kpt);
    }
    gl.tiles = ktiles;  // reused as k tiles
    const int64_t ctas = rows * ktiles;
    int64_t nbs = 1;
    if (ctas < target && nb > 1) nbs = std::min<int64_t>(nb, (target + ctas - 1) / ctas);
    gl.bper = int((nb + nbs - 1) / nbs);
    gl.nbs = int((nb + gl.bper - 1) / gl.bper);
    gl.mode = (t.all_gemm && 8ll * t.C * (gl.bper + 1) <= 96 * 1024) ? 0 : 2;
    return gl;
  }
  // warp-specialised grid kernel: (row, batch slab, k tile) tiles.  With few
  // rows, row-block (general-mode) grids split the k axis first (>= 256 k
  // per tile): a tile then resolves each k once for its whole batch slab
  const int64_t target_tiles = 148 * 8;
  int64_t nbs = 1;
  const bool k_first = !t.all_gemm && rows < target_tiles;
  if (k_first) {
    const int64_t nkt_max = std::max<int64_t>(1, g.nK / kConsumers);
    const int64_t per_row = (target_tiles + rows - 1) / rows;
    if (per_row > nkt_max && nb > 1)
      nbs = std::min<int64_t>(nb, (per_row + nkt_max - 1) / nkt_max);
  } else if (rows < target_tiles && nb > 1) {
    nbs = std::min<int64_t>(nb, (target_tiles + rows - 1) / rows);
  }
  gl.bper = int((nb + nbs - 1) / nbs);
  gl.nbs = int((nb + gl.bper - 1) / gl.bper);
  // too few (row, slab) tiles (attention grids: one (m, n) row, long k axis):
  // split the k axis too, >= 1024 k values per tile
  gl.nkt = 1;
  gl.kt = int(g.nK);
  const int64_t min_kt = k_first ? kConsumers : 1024;
  if (rows * gl.nbs < target_tiles && g.nK > min_kt)
    gl.nkt = int(std::min<int64_t>((target_tiles + rows * gl.nbs - 1) / (rows * gl.nbs),
                                   (g.nK + min_kt - 1) / min_kt));
  if (gl.nkt > 1) {
    gl.kt = int((g.nK + gl.nkt - 1) / gl.nkt);
    gl.nkt = int((g.nK + gl.kt - 1) / gl.kt);
  }
  gl.tiles = int(std::min<int64_t>(rows * gl.nbs * std::max(gl.nkt, 1), 0x7FFFFFFFll));
  gl.kpt = int((g.nK + kConsumers - 1) / kConsumers);
  gl.mode = t.all_gemm ? 0 : 2;
  gl.near = (t.NC == 1 && t.lowest_wins) ? 2 : (t.G <= 32 ? 1 : 0);
  smem_layout(t, gl);
  if (gl.mode == 0 && gl.smem > 160 * 1024) {  // W slices too large for smem
    gl.mode = 1;
    smem_layout(t, gl);
  }
  gl.ctas = int(std::min<int64_t>(gl.tiles, 148 * 3));
  return gl;
}

// The one-class lookup kernel applies to latency-only launches of GEMM grids
// whose tables form one member class, with an even k axis (16-byte pair
// stores into a 16-byte aligned output) and u8-sized staircases; rl.tiles
// == 0 otherwise.
RowLaunch plan_rows(const TablesDev& t, const GridDev& g, const GridLaunch& gl,
                    const LaunchOut& out, int* nb_out) {
  RowLaunch rl{};
  const int64_t nb = g.b_hi - g.b_lo;
  if (std::getenv("PM2L_DEBUG_PLAN"))  // diagnostics
    std::fprintf(stderr,
                 "plan_rows: curve=%d near=%d all_gemm=%d kfast=%d nK=%lld nb=%lld align=%d CM=%d G=%d "
                 "NW=%d cm_tab=%d\n",
                 out.curve != nullptr, gl.near, t.all_gemm, g.kfast != nullptr, (long long)g.nK,
                 (long long)nb, int(reinterpret_cast<uintptr_t>(out.lat) & 15), t.CM, t.G, t.NW,
                 g.cm_tab != nullptr);
  if (out.curve || gl.near != 2 || !(t.all_gemm || t.all_rowblock) || !g.kfast || nb <= 0 ||
      t.CM > 254 || t.CM < 1 || g.nM * g.nN > 0x7FFFFFFFll)
    return rl;
  rl.pair = g.nK % 2 == 0 && (reinterpret_cast<uintptr_t>(out.lat) & 15) == 0;
  rl.rowblock = t.all_rowblock;
  if (rl.rowblock && !rl.pair) return rl;  // row-block variant: pair stores only
  if ((t.all_gemm && !g.cm_tab) || t.NW < 1) return rl;
  int NB = 8;
  while (nb % NB) NB >>= 1;
  rl.kc = int(std::min<int64_t>(g.nK, kKChunk));
  rl.nkc = int((g.nK + rl.kc - 1) / rl.kc);
  // few (m, n) rows (attention grids: one row, long k): narrower batch slabs
  // until every CTA slot has about two tiles, since a tile's emission is
  // latency-bound on its 4 writer warps
  while (NB > 1 && g.nM * g.nN * (nb / NB) * rl.nkc < 2 * 148 * 3) NB >>= 1;
  if (const char* e = std::getenv("PM2L_ROW_NB")) {  // experiments
    const int v = std::atoi(e);
    if (v >= 1 && v <= 8 && (v & (v - 1)) == 0 && nb % v == 0) NB = v;
  }
  rl.nbs = int(nb / NB);
  rl.d_nkc = fast_div_for(uint32_t(rl.nkc));
  rl.d_nbs = fast_div_for(uint32_t(rl.nbs));
  rl.d_nN = fast_div_for(uint32_t(g.nN));
  const bool stage_k = g.nK <= kKChunk;
  rl.ring = 1;
  rl.prod = kRingProd;
  rl.slots = kRingSlots;
  if (const char* e = std::getenv("PM2L_ROW_RING")) rl.ring = std::atoi(e);  // experiments
  if (const char* e = std::getenv("PM2L_RING_PROD")) rl.prod = std::min(std::max(std::atoi(e), 1), kRowWarps - 1);
  if (const char* e = std::getenv("PM2L_RING_SLOTS")) rl.slots = std::min(std::max(std::atoi(e), 1), kRingMaxSlots);
  const int64_t tiles = g.nM * g.nN * rl.nbs * rl.nkc;
  if (tiles > 0x7FFFFFFFll || t.G + t.CM > 4096) return rl;
  row_layout(t, g, NB, stage_k, rl);
  if (std::getenv("PM2L_DEBUG_PLAN"))
    std::fprintf(stderr, "plan_rows: smem=%lld tiles=%lld\n", (long long)rl.smem, (long long)tiles);
  if (rl.smem > 200 * 1024) return rl;
  rl.tiles = int(tiles);
  rl.ctas = int(std::min<int64_t>((tiles + kRowWarps - 1) / kRowWarps, 148 * 3));
  if (rl.rowblock && !rl.ring) return RowLaunch{};  // row-block: ring kernel only
  if (rl.ring) rl.ctas = int(std::min<int64_t>(tiles, 148 * 3));
  if (const char* e = std::getenv("PM2L_ROW_CTAS")) {  // tuning experiments only
    const int v = std::atoi(e);
    if (v > 0) rl.ctas = std::min(rl.ctas, v);
  }
  *nb_out = NB;
  return rl;
}

template <int NB, bool STAGE, int SEGW>
cudaError_t launch_rows_k(const TablesDev& t, const GridDev& g, const RowLaunch& rl,
                          const double* base, const LaunchOut& out, cudaStream_t s) {
  auto* fn = rl.rowblock ? grid_ring_kernel<NB, STAGE, SEGW, true, true>
             : rl.pair ? (rl.ring ? grid_ring_kernel<NB, STAGE, SEGW, true, false>
                                  : grid_row_kernel<NB, STAGE, SEGW, true>)
                       : (rl.ring ? grid_ring_kernel<NB, STAGE, SEGW, false, false>
                                  : grid_row_kernel<NB, STAGE, SEGW, false>);
  if (rl.smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rl.smem));
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(rl.ctas));
  cfg.blockDim = dim3(32 * kRowWarps);
  cfg.dynamicSmemBytes = size_t(rl.smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, t, g, rl, base, out);
}

template <int NB>
cudaError_t launch_rows_t(const TablesDev& t, const GridDev& g, const RowLaunch& rl,
                          const double* base, const LaunchOut& out, cudaStream_t s) {
  const bool stage = g.nK <= kKChunk;
  if (rl.seg == 16)
    return stage ? launch_rows_k<NB, true, 4>(t, g, rl, base, out, s)
                 : launch_rows_k<NB, false, 4>(t, g, rl, base, out, s);
  if (rl.seg == 32)
    return stage ? launch_rows_k<NB, true, 8>(t, g, rl, base, out, s)
                 : launch_rows_k<NB, false, 8>(t, g, rl, base, out, s);
  return stage ? launch_rows_k<NB, true, 16>(t, g, rl, base, out, s)
               : launch_rows_k<NB, false, 16>(t, g, rl, base, out, s);
}

bool grid_dims_ok(const GridDev& g, const GridLaunch& gl) {
  return g.nM * g.nN * gl.nbs * std::max(gl.nkt, 1) <= 0x7FFFFFFFll && gl.nbs <= 65535 && g.nK <= 0x3FFFFFFFll &&
         g.nB <= 0x7FFFFFFFll;
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

void launch_base_table(const TablesDev& t, const GridDev& g, double* ws, double* fixval,
                       unsigned long long* stats, cudaStream_t s) {
  const int chunks = int(std::min<int64_t>((g.nK + 255) / 256, 64));
  const int ys = std::max(1, t.C + (fixval && g.n_fix > 0 ? 1 : 0));
  base_table_kernel<<<dim3(chunks, ys), 256, 0, s>>>(t, g, g.K, int(g.nK), ws, fixval, stats);
}

}  // namespace

int64_t grid_workspace_elems(const TablesDev& t, const GridDev& g) {
  return int64_t(t.C) * g.nK + g.n_fix;  // base table, then exact-hit values
}

int grid_kernel_path(const TablesDev& t, const GridDev& g, const LaunchOut& out) {
  const GridLaunch gl = plan_grid(t, g, false);
  int nb = 0;
  return plan_rows(t, g, gl, out, &nb).tiles > 0 ? 3 : gl.near;
}

int launch_grid(const TablesDev& t, const GridDev& g, int64_t /*max_group*/, double* ws,
                int64_t ws_elems, const LaunchOut& out, void* stream, int stages) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t card = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  if (card == 0) return 0;
  const GridLaunch gl = plan_grid(t, g, false);
  const int64_t nbase = int64_t(t.C) * g.nK, need = nbase + g.n_fix;
  if ((need > 0 && (!ws || ws_elems < need)) || !grid_dims_ok(g, gl) || gl.smem > 227 * 1024 ||
      t.C >= 65535 || nbase > 0x7FFFFFFFll)
    return int(cudaErrorInvalidValue);
  const double* base = t.C > 0 ? ws : nullptr;
  // exact-hit values are precomputed with the base table whenever it runs in
  // the same launch sequence (stage masks that skip it recompute in fixup_kernel)
  double* fixval = (g.n_fix > 0 && (stages & kStageBase)) ? ws + nbase : nullptr;
  if (stages & kStageBase) launch_base_table(t, g, ws, fixval, out.nan_stats, s);
  const bool v = out.curve != nullptr;
  cudaError_t e = cudaSuccess;
  int row_nb = 0;
  const RowLaunch rl = plan_rows(t, g, gl, out, &row_nb);
  if ((stages & kStageGrid) && rl.tiles > 0) {
    e = row_nb == 8   ? launch_rows_t<8>(t, g, rl, base, out, s)
        : row_nb == 4 ? launch_rows_t<4>(t, g, rl, base, out, s)
        : row_nb == 2 ? launch_rows_t<2>(t, g, rl, base, out, s)
                      : launch_rows_t<1>(t, g, rl, base, out, s);
  } else if (stages & kStageGrid) {
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
  // the row kernel applies its rows' exact hits itself
  const bool fixed_in_grid = (stages & kStageGrid) && rl.tiles > 0;
  if (g.n_fix > 0 && (stages & kStageFixup) && !fixed_in_grid) {
    const int nb = int((g.n_fix + 127) / 128);
    if (v) fixup_kernel<true><<<nb, 128, 0, s>>>(t, g, out, nullptr);
    else fixup_kernel<false><<<nb, 128, 0, s>>>(t, g, out, fixval);
  }
  return int(cudaGetLastError());
}

int launch_grid_all_curves(const TablesDev& t, const GridDev& g, double* ws, double* out,
                           void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t card = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  if (card == 0 || t.C == 0) return 0;
  GridLaunch gl = plan_grid(t, g, true);
  if (!grid_dims_ok(g, gl) || t.C > 65535 || gl.tiles > 65535) return int(cudaErrorInvalidValue);
  launch_base_table(t, g, ws, nullptr, nullptr, s);
  const int64_t smem = gl.mode == 0 ? ((8ll * t.C + 15) & ~15ll) + 8ll * t.C * gl.bper : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(all_curves_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return int(e);
  }
  const dim3 grid(unsigned(g.nM * g.nN), unsigned(gl.tiles), unsigned(gl.nbs));
  all_curves_kernel<<<grid, kThreads, smem, s>>>(t, g, gl, ws, out);
  return int(cudaGetLastError());
}

#ifdef PM2L_TIMING
int row_timing_copy(unsigned long long* host, int n) {
  if (n < 0) return int(cudaMemcpyFromSymbol(host, g_pdl_dbg, sizeof(unsigned long long) * size_t(-n)));
  return int(cudaMemcpyFromSymbol(host, g_row_dbg, sizeof(unsigned long long) * size_t(n)));
}
#endif

int launch_nan_scan(const double* v, int64_t n, unsigned long long* first, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
  nan_scan_kernel<<<nb, 256, 0, s>>>(v, n, first);
  return int(cudaGetLastError());
}

}  // namespace pm2l
