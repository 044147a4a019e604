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
#include "grid_common.cuh"

namespace pm2l {
namespace gk {
namespace {

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

// Exact-record hits take priority over the nearest result (_kernels.pyx:107-110).
// `fixval` (nullable) holds their latencies, precomputed by the base-table
// kernel off the critical path.
template <bool VERIFY>
__global__ void fixup_kernel(TablesDev t, GridDev g, LaunchOut out, const double* fixval) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= g.n_fix) return;
  const int64_t p = g.fix_pos[i];
  if (p < 0) return;  // device plans: a record off this slice
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
  if (gl.kt == 2 && table) {
    // two adjacent k per thread, one 16-byte streaming store per (curve,
    // batch value): even k axis, 16-byte aligned output (plan_grid)
    // curve-major: a CTA writes each (curve, batch value) run of its k tile
    // back to back (longer contiguous DRAM runs than k-major order)
    const int p0 = int(blockIdx.y) * gl.kpt * int(blockDim.x);
    const int ik0 = 2 * (p0 + tid);
    for (int c = 0; c < t.C; ++c) {
      const bool valid = curve_valid(t, c);
      double2 base[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ik = ik0 + 2 * j * int(blockDim.x);
        base[j] = j < gl.kpt && ik < nK ? *reinterpret_cast<const double2*>(base_tab + int64_t(c) * nK + ik)
                                        : make_double2(0.0, 0.0);
      }
      double* o = out + int64_t(c) * slice + row_off + ik0;
      for (int ib = 0; ib < nb; ++ib, o += plane) {
        const double w = W[ib * t.C + c];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ik = ik0 + 2 * j * int(blockDim.x);
          if (j < gl.kpt && ik < nK) {
            const double2 lat = valid ? make_double2(__dmul_rn(base[j].x, w), __dmul_rn(base[j].y, w))
                                      : make_double2(qnan(), qnan());
            __stcs(reinterpret_cast<double2*>(o + 2 * j * int(blockDim.x)), lat);
          }
        }
      }
    }
    return;
  }
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

GridLaunch plan_grid(const TablesDev& t, const GridDev& g, bool all_curves, bool aligned16 = false) {
  GridLaunch gl{};
  const int64_t rows = g.nM * g.nN;
  const int64_t nb = g.b_hi - g.b_lo;
  if (all_curves) {  // all_curves_kernel: (row, k tile, slab) CTAs of kThreads
    const int64_t target = int64_t(sm_count()) * 8;
    // kt: k values per thread step (2: 16-byte pair stores on an even k
    // axis; needs the W table, which the condition below guarantees: mode 0)
    gl.kt = aligned16 && g.nK % 2 == 0 && t.all_gemm && (8ll * t.C * (nb + 1) <= 96 * 1024) ? 2 : 1;
    auto ktiles_for = [&](int kpt) {
      const int64_t per = int64_t(kpt) * kThreads * gl.kt;
      return int((g.nK + per - 1) / per);
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
  const int64_t target_tiles = int64_t(sm_count()) * 8;
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
  gl.ctas = int(std::min<int64_t>(gl.tiles, int64_t(sm_count()) * kSweepCtasPerSm));
  return gl;
}

#ifdef PM2L_TIMING
// diagnostic build only: device buffers of the per-tile / per-CTA stamps
}  // namespace
unsigned long long** timing_buffers() {
  static unsigned long long* b[2] = {nullptr, nullptr};
  if (!b[0]) {
    cudaMalloc(&b[0], sizeof(unsigned long long) * 16384 * 8);
    cudaMalloc(&b[1], sizeof(unsigned long long) * 4096 * 4);
  }
  return b;
}
namespace {
#endif

// Launch-shape overrides for tuning experiments (tools/ab_*.sh), read once
// per process -- never on the launch path.  PM2L_DEBUG_PLAN prints the plan.
struct Tuning {
  int nb = 0, prod = 0, slots = 0, ctas = 0;
  bool debug = false;
};
const Tuning& tuning() {
  static const Tuning k = [] {
    Tuning t;
    auto geti = [](const char* name) {
      const char* e = std::getenv(name);
      return e ? std::atoi(e) : 0;
    };
    t.nb = geti("PM2L_ROW_NB");
    t.prod = geti("PM2L_RING_PROD");
    t.slots = geti("PM2L_RING_SLOTS");
    t.ctas = geti("PM2L_ROW_CTAS");
    t.debug = std::getenv("PM2L_DEBUG_PLAN") != nullptr;
    return t;
  }();
  return k;
}

// The one-class lookup kernel applies to latency-only launches of GEMM grids
// whose tables form one member class, with an even k axis (16-byte pair
// stores into a 16-byte aligned output) and u8-sized staircases; rl.tiles
// == 0 otherwise.
RowLaunch plan_rows(const TablesDev& t, const GridDev& g, const GridLaunch& gl,
                    const LaunchOut& out, int* nb_out) {
  RowLaunch rl{};
  const Tuning& tu = tuning();
  const int64_t nb = g.b_hi - g.b_lo;
  const int64_t slots_total = int64_t(sm_count()) * kRowCtasPerSm;
  if (tu.debug)
    std::fprintf(stderr,
                 "plan_rows: curve=%d near=%d all_gemm=%d kfast=%d nK=%lld nb=%lld align=%d CM=%d G=%d "
                 "NW=%d k_sorted=%d\n",
                 out.curve != nullptr, gl.near, t.all_gemm, g.kfast != nullptr, (long long)g.nK,
                 (long long)nb, int(reinterpret_cast<uintptr_t>(out.lat) & 15), t.CM, t.G, t.NW,
                 g.k_sorted);
  // the byte maps and per-chunk group cuts assume an ascending k axis (the
  // canonical GridSpec order); the raw FFI accepts any order, which takes
  // the order-independent sweep kernel
  if (out.curve || gl.near != 2 || !(t.all_gemm || t.all_rowblock) || !g.kfast || !g.k_sorted ||
      nb <= 0 || t.CM > 254 || t.CM < 1 || g.nM * g.nN > 0x7FFFFFFFll)
    return rl;
  rl.pair = g.nK % 2 == 0 && (reinterpret_cast<uintptr_t>(out.lat) & 15) == 0;
  rl.rowblock = t.all_rowblock;
  if (rl.rowblock && !rl.pair) return rl;  // row-block variant: pair stores only
  if (t.NW < 1) return rl;
  int NB = 8;
  while (nb % NB) NB >>= 1;
  rl.kc = int(std::min<int64_t>(g.nK, kKChunk));
  rl.nkc = int((g.nK + rl.kc - 1) / rl.kc);
  // few (m, n) rows (attention grids: one row, long k): narrower batch slabs
  // until every CTA slot has about two tiles, since a tile's emission is
  // latency-bound on its 4 writer warps
  while (NB > 1 && g.nM * g.nN * (nb / NB) * rl.nkc < 2 * slots_total) NB >>= 1;
  if (tu.nb >= 1 && tu.nb <= 8 && (tu.nb & (tu.nb - 1)) == 0 && nb % tu.nb == 0) NB = tu.nb;
  rl.nbs = int(nb / NB);
  rl.d_nkc = fast_div_for(uint32_t(rl.nkc));
  rl.d_nbs = fast_div_for(uint32_t(rl.nbs));
  rl.d_nN = fast_div_for(uint32_t(g.nN));
  const bool stage_k = g.nK <= kKChunk;
  // rank/group byte maps per tile (GEMM grids: many rows share the k
  // ranks, a map serves NB batch values) or the per-k closed-form resolve
  // (row-block grids: one (m, n) row and a long k axis, where the planner's
  // k ranks would dominate a plan-inclusive launch)
  // (device code keys the variant on the row-block template parameter)
  rl.direct = t.all_rowblock ? 1 : 0;
  rl.prod = tu.prod > 0 ? std::min(tu.prod, kRowWarps - 1) : kRingProd;
  rl.slots = tu.slots > 0 ? std::min(tu.slots, kRingMaxSlots) : stage_k ? kRingSlotsStaged : kRingSlots;
  const int64_t tiles = g.nM * g.nN * rl.nbs * rl.nkc;
  if (tiles > 0x7FFFFFFFll || t.G + t.CM > 4096) return rl;
  row_layout(t, g, NB, stage_k, rl);
  if (tu.debug)
    std::fprintf(stderr, "plan_rows: smem=%lld tiles=%lld\n", (long long)rl.smem, (long long)tiles);
  if (rl.smem > 200 * 1024) return rl;
  rl.tiles = int(tiles);
  rl.ctas = int(std::min<int64_t>(tiles, slots_total));
  if (tu.ctas > 0) rl.ctas = std::min(rl.ctas, tu.ctas);
#ifdef PM2L_TIMING
  rl.dbg_row = timing_buffers()[0];
  rl.dbg_pdl = timing_buffers()[1];
#endif
  *nb_out = NB;
  return rl;
}

bool grid_dims_ok(const GridDev& g, const GridLaunch& gl) {
  return g.nM * g.nN * gl.nbs * std::max(gl.nkt, 1) <= 0x7FFFFFFFll && gl.nbs <= 65535 && g.nK <= 0x3FFFFFFFll &&
         g.nB <= 0x7FFFFFFFll;
}

void launch_base_table(const TablesDev& t, const GridDev& g, double* ws, double* fixval,
                       unsigned long long* stats, cudaStream_t s) {
  const int chunks = int(std::min<int64_t>((g.nK + 255) / 256, 64));
  const int ys = std::max(1, t.C + (fixval && g.n_fix > 0 ? 1 : 0));
  base_table_kernel<<<dim3(chunks, ys), 256, 0, s>>>(t, g, g.K, int(g.nK), ws, fixval, stats);
}

}  // namespace
}  // namespace gk

using namespace gk;

int64_t grid_workspace_elems(const TablesDev& t, const GridDev& g) {
  return int64_t(t.C) * g.nK + g.n_fix;  // base table, then exact-hit values
}

int grid_kernel_path(const TablesDev& t, const GridDev& g, const LaunchOut& out) {
  if (single_ok(t, g, out)) return 4;
  const GridLaunch gl = plan_grid(t, g, false);
  int nb = 0;
  return plan_rows(t, g, gl, out, &nb).tiles > 0 ? 3 : gl.near;
}

int launch_grid(const TablesDev& t, const GridDev& g, int64_t /*max_group*/, double* ws,
                int64_t ws_elems, const LaunchOut& out, void* stream, int stages) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t card = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  if (card == 0) return 0;
  // single-member tables: one planner-free kernel (its exact hits inline)
  if (single_ok(t, g, out)) return int(launch_single(t, g, out, stages, s));
  const GridLaunch gl = plan_grid(t, g, false);
  const int64_t nbase = int64_t(t.C) * g.nK, need = nbase + g.n_fix;
  if ((need > 0 && (!ws || ws_elems < need)) || !grid_dims_ok(g, gl) || gl.smem > 227 * 1024 ||
      t.C >= 65535 || nbase > 0x7FFFFFFFll)
    return int(cudaErrorInvalidValue);
  const double* base = t.C > 0 ? ws : nullptr;
  // exact-hit values are precomputed with the base table whenever it runs in
  // the same launch sequence (stage masks that skip it, and device-planned
  // slices, recompute them in fixup_kernel)
  double* fixval = (g.n_fix > 0 && (stages & kStageBase) && !g.dev_planned) ? ws + nbase : nullptr;
  int row_nb = 0;
  const RowLaunch rl = plan_rows(t, g, gl, out, &row_nb);
  if (stages & kStageBase) {
    if (g.dev_planned) {
      // the k ranks only feed the lookup kernel's byte maps
      const bool ranks = rl.tiles > 0 && !rl.direct;
      if (const int rc = launch_dplan(t, g, ws, out.nan_stats, ranks, s)) return rc;
    } else {
      launch_base_table(t, g, ws, fixval, out.nan_stats, s);
    }
  }
  const bool v = out.curve != nullptr;
  cudaError_t e = cudaSuccess;
  if ((stages & kStageGrid) && rl.tiles > 0) {
    GridDev gr = g;
    gr.plan_ready = g.dev_planned && !(stages & kStageBase);
    e = row_nb == 8   ? launch_rows_t<8>(t, gr, rl, base, out, s)
        : row_nb == 4 ? launch_rows_t<4>(t, gr, rl, base, out, s)
        : row_nb == 2 ? launch_rows_t<2>(t, gr, rl, base, out, s)
                      : launch_rows_t<1>(t, gr, rl, base, out, s);
  } else if (stages & kStageGrid) {
    e = launch_sweep(t, g, gl, base, out, s);
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
  GridLaunch gl = plan_grid(t, g, true, (reinterpret_cast<uintptr_t>(out) & 15) == 0);
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
  unsigned long long** buf = gk::timing_buffers();
  if (n < 0) return int(cudaMemcpy(host, buf[1], sizeof(unsigned long long) * size_t(-n), cudaMemcpyDeviceToHost));
  return int(cudaMemcpy(host, buf[0], sizeof(unsigned long long) * size_t(n), cudaMemcpyDeviceToHost));
}
#endif

int launch_nan_scan(const double* v, int64_t n, unsigned long long* first, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + 255) / 256, int64_t(sm_count()) * 16));
  nan_scan_kernel<<<nb, 256, 0, s>>>(v, n, first);
  return int(cudaGetLastError());
}

}  // namespace pm2l