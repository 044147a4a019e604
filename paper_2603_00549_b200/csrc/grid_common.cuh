// Grid-mode launch descriptors and device helpers shared by the grid
// translation units (grid.cu: planning + small kernels; grid_sweep.cu: the
// general k-group sweep kernel; grid_lookup_nb*.cu: the one-class lookup
// kernel, one batch-slab width per unit so they compile in parallel).
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace pm2l {
namespace gk {

using namespace dev;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;"); }

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

constexpr int kRowWarps = 8;
constexpr int kRingProd = 4;   // grid_ring_kernel: default builder warps per CTA
constexpr int kRingSlots = 6;  // default tile-state slots per CTA (k axes longer than a chunk)
constexpr int kRingSlotsStaged = 4;  // k axis in one staged chunk (C2 sweep of 3 / 4 / 5 / 6 / 8)
constexpr int kRingMaxSlots = 16;
constexpr int kRowCtasPerSm = 3;    // __launch_bounds__ minimum of grid_ring_kernel
constexpr int kSweepCtasPerSm = 3;

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
  int pair;                  // 16-byte pair stores (even k axis, aligned output)
  int rowblock;              // row-block tables: per-point wave scale (ring kernel, pairs)
  int prod, slots;           // ring: builder warps, tile-state slots
  int direct;                // per-k closed-form resolve (no byte maps, no k ranks)
  int ctas;
  int off_bar, off_gcur, off_glk, off_clm, off_cln, off_wcp, off_kf, off_ms, off_kq, off_kr, off_ki,
      off_warp;
  int w_hdr, w_sD, w_sP, w_cut, w_W, w_rmap, w_gmap, warp_bytes;
  int64_t smem;
#ifdef PM2L_TIMING
  unsigned long long* dbg_row;  // diagnostic build: per-tile phase stamps
  unsigned long long* dbg_pdl;  // per CTA: entry, before/after pdl wait, first FULL
#endif
};

inline void row_layout(const TablesDev& t, const GridDev& g, int nb, bool stage_k, RowLaunch& rl) {
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
  const bool maps = !rl.direct;
  rl.off_kf = take(stage_k && maps ? 4ll * g.nK : 0);
  rl.off_ms = take(stage_k && maps ? 8ll * g.nK : 0);
  rl.off_kq = take(stage_k && maps ? 8ll * g.nK : 0);
  rl.off_kr = take(stage_k && maps ? 4ll * rl.nkc * t.G : 0);
  rl.off_ki = take(stage_k && !maps ? int64_t(sizeof(KInfo)) * g.nK : 0);
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
  rl.w_cut = wtake(maps ? 4ll * (t.CM + t.G + 1) : 0);
  rl.w_W = wtake(8ll * t.NW * nb);
  rl.w_rmap = wtake(maps ? 32ll * rl.seg : 0);
  rl.w_gmap = wtake(maps ? 32ll * rl.seg : 0);
  rl.warp_bytes = int(w);
  rl.smem = o + int64_t(rl.slots) * w;
}

#ifdef PM2L_TIMING
unsigned long long** timing_buffers();  // grid.cu: [0] per-tile rows, [1] per-CTA stamps
#endif
// single-member tables (grid_single.cu): no planner, no tile builds
bool single_ok(const TablesDev& t, const GridDev& g, const LaunchOut& out);
cudaError_t launch_single(const TablesDev& t, const GridDev& g, const LaunchOut& out, int stages,
                          cudaStream_t s);
// general k-group sweep kernel (grid_sweep.cu)
cudaError_t launch_sweep(const TablesDev& t, const GridDev& g, const GridLaunch& gl,
                         const double* base, const LaunchOut& out, cudaStream_t s);
// one-class lookup kernel for NB batch values per tile (grid_lookup_nb<NB>.cu)
template <int NB>
cudaError_t launch_rows_t(const TablesDev& t, const GridDev& g, const RowLaunch& rl,
                          const double* base, const LaunchOut& out, cudaStream_t s);
extern template cudaError_t launch_rows_t<1>(const TablesDev&, const GridDev&, const RowLaunch&,
                                             const double*, const LaunchOut&, cudaStream_t);
extern template cudaError_t launch_rows_t<2>(const TablesDev&, const GridDev&, const RowLaunch&,
                                             const double*, const LaunchOut&, cudaStream_t);
extern template cudaError_t launch_rows_t<4>(const TablesDev&, const GridDev&, const RowLaunch&,
                                             const double*, const LaunchOut&, cudaStream_t);
extern template cudaError_t launch_rows_t<8>(const TablesDev&, const GridDev&, const RowLaunch&,
                                             const double*, const LaunchOut&, cudaStream_t);

}  // namespace gk
}  // namespace pm2l
