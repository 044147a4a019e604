// One-class lookup kernel (grid_ring_kernel) of the grid mode.  Included by
// grid_lookup_nb<NB>.cu, each instantiating launch_rows_t<NB>.
#pragma once

#include "grid_common.cuh"

namespace pm2l {
namespace gk {

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

#ifdef PM2L_TIMING
// diagnostic build only (tools/row_timing.py): per-tile phase timestamps
#define ROW_MARK(tile, i)                                                         \
  do {                                                                            \
    if (lane == 0 && (tile) < 16384) {                                            \
      rl.dbg_row[(tile) * 8 + (i)] = clock64();                                   \
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
  uint64_t m, n;  // the row's shape (W table: tile counts per wave class)
};

template <int NB, bool RB = false>
__device__ __forceinline__ RowIn<NB> load_row_in(const GridDev& g, const RowLaunch& rl, int tile,
                                                 int NW, int lane) {
  RowIn<NB> r;
  const int rs = fdiv(tile, rl.d_nkc), row = fdiv(rs, rl.d_nbs), slab = rs - row * rl.nbs;
  const int im = fdiv(row, rl.d_nN), jn = row - im * int(g.nN);
  r.im = im;
  r.jn = jn;
  r.m = g.M[im];
  r.n = g.N[jn];
  if (g.lut) {
    // device plans: the row's log2 straight from the per-device libm table,
    // so a tile's staircase and W table never wait for the planner kernel
    // (an out-of-range value is the planner's reported contract violation)
    r.qm = r.m < uint64_t(g.lut_n) ? g.lut[r.m] : 0.0;
    r.qn = r.n < uint64_t(g.lut_n) ? g.lut[r.n] : 0.0;
  } else {
    r.qm = g.logM[im];
    r.qn = g.logN[jn];
  }
#pragma unroll
  for (int ib = 0; ib < NB; ++ib) r.b[ib] = g.B[g.b_lo + slab * NB + ib];
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
  const KInfo* ki;       // direct resolve: {log2 k, k-group insertion point} per k
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
  c.ki = STAGE ? reinterpret_cast<const KInfo*>(smem + rl.off_ki) : g.kinfo;
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
}

// The per-k tables of the slice (STAGE): on bar + 1.  A device-planned
// slice's come from the planner kernel, so the issuing thread has passed
// griddepcontrol.wait first.
template <bool STAGE>
__device__ __forceinline__ void row_prologue_k(uint8_t* smem, const RowCtx<STAGE>& c,
                                               const GridDev& g, const RowLaunch& rl, uint64_t* bar) {
  if (rl.direct) {
    mbar_expect_tx(bar + 1, r16(int64_t(sizeof(KInfo)) * c.nK));
    bulk_g2s(smem + rl.off_ki, g.kinfo, r16(int64_t(sizeof(KInfo)) * c.nK), bar + 1);
    return;
  }
  mbar_expect_tx(bar + 1, r16(4ll * c.nK) + 2 * r16(8ll * c.nK) + r16(4ll * rl.nkc * c.G));
  bulk_g2s(smem + rl.off_ms, g.mn_sorted, r16(8ll * c.nK), bar + 1);
  bulk_g2s(smem + rl.off_kq, g.logK, r16(8ll * c.nK), bar + 1);
  bulk_g2s(smem + rl.off_kr, g.kright, r16(4ll * rl.nkc * c.G), bar + 1);
  bulk_g2s(smem + rl.off_kf, g.kfast, r16(4ll * c.nK), bar + 1);
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
    // ceil(m / tile_m) * ceil(n / tile_n) * split_k in u64 (the reference's
    // block product, _kernels.pyx:126; wrapping like the host planner's)
    const uint64_t tmn = ceil_div_w(p, 0, cur.m, p.tm) * (ceil_div_w(p, 1, cur.n, p.tn) * p.sk);
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
                                           uint64_t* stair_ready = nullptr,
                                           uint64_t* k_ready = nullptr, bool plan_wait = false) {
  // k_ready / plan_wait (a builder's first tile): the staircase and W table
  // need only the CTA tables; the cut searches below also need the slice's
  // per-k tables (bar k_ready) and, for device plans, the planner kernel
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
  if (RB) {  // row-block tables resolve per k in closed form (rl.direct)
    // per-k closed form at emission: the tile state is the staircase, its
    // minimum and first minimiser, and the W table
    if (lane == 0) {
      hdr[0] = len;
      hdr[1] = lastpos;
      *reinterpret_cast<uint64_t*>(hdr + 2) = dmin;
    }
    return;
  }
  if (plan_wait) pdl_wait();
  if (STAGE && k_ready) mbar_wait(k_ready, 0);
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
  // direct: nearest_one_class (grid_sweep.cu) per k from {log2 k, insertion
  // point}: the nearest k-groups' distance mn decides case A (mn <= dmin:
  // leftmost group within dmin, member lastpos) or case B (leftmost group
  // at mn, member = first staircase step <= mn); same comparisons, same bits
  const uint64_t* sD = reinterpret_cast<const uint64_t*>(wb + rl.w_sD);
  const uint64_t dmin = *reinterpret_cast<const uint64_t*>(hdr + 2);
  const int len = hdr[0];
  int top = 1;
  while (top * 2 <= len) top *= 2;
  auto resolve = [&](const KInfo& q) -> int2 {
    const double qk = q.qk;
    const int start = q.start, G = c.G;
    auto dk = [&](int gg) { return abs_bits(__dsub_rn(c.glk[gg], qk)); };
    const uint64_t dkL = start > 0 ? dk(start - 1) : ~0ull;
    const uint64_t dkR = start < G ? dk(start) : ~0ull;
    const uint64_t mn = dkL < dkR ? dkL : dkR;
    const bool case_a = mn <= dmin;
    const uint64_t lim = case_a ? dmin : mn;  // walk left while within it (A) / tied (B)
    int gg = start;
    if (case_a ? dkL <= dmin : dkL == mn) {
      gg = start - 1;
      while (gg > 0 && (case_a ? dk(gg - 1) <= lim : dk(gg - 1) == lim)) --gg;
    }
    int pos = lastpos;
    if (!case_a) {  // #{steps with sD > mn} (sD strictly descends; sD[len-1] = dmin < mn)
      int s = 0;
      for (int step = top; step; step >>= 1)
        if (s + step <= len && sD[s + step - 1] > mn) s += step;
      pos = sP[s];
    }
    return c.gcur[gg * CM + pos];
  };
  constexpr int U = 4;
  for (int bq = b0; bq < nB; bq += U * bstep) {  // warp-uniform trip count (__all_sync)
    int2 v[U][2];
    int pp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      pp[u] = (bq + u * bstep) * 32 + lane;
      const int p = min(pp[u], nP - 1);
      if (RB) {  // compile-time: the GEMM emission loop carries no direct-resolve code
        v[u][0] = resolve(c.ki[k0 + 2 * p]);
        v[u][1] = has_second(p) ? resolve(c.ki[k0 + 2 * p + 1]) : v[u][0];
      } else {
        const uint2 kf = *reinterpret_cast<const uint2*>(c.kfs + k0 + 2 * p);
        v[u][0] = lookup(kf.x, 2 * p);
        v[u][1] = has_second(p) ? lookup(kf.y, 2 * p + 1) : v[u][0];
      }
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
  int f0, f1;
  if (g.fixr_rng) {  // device plan: the row's record range (off-slice entries skip below)
    const int2 fr = g.fixr_rng[x.row];
    f0 = fr.x;
    f1 = fr.y;
  } else {
    f0 = g.fixr_off[x.row];
    f1 = g.fixr_off[x.row + 1];
  }
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
        // the record's curve: base(curve, k) x the wave scale of its wave
        // class for this batch value -- the tile's W table (GEMM), or the
        // row-block scale from the staged class parameters: no dependent
        // global loads on a tile's last writer
        const double bse = base_tab[ci * nK + fe.ik];
        const int ibl = fe.ib - x.slab * NB;
        if (RB) {
          const uint64_t b = uint64_t(__double_as_longlong(W[ibl]));
          *o = __dmul_rn(bse, rb_scale(c.wcp[fe.wc], b, g.K[fe.ik]));
        } else {
          *o = __dmul_rn(bse, W[fe.wc * NB + ibl]);
        }
      }
    }
  }
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
    // host plans (and device plans completed by an earlier launch): the
    // per-k tables are ready now; device plans of this launch sequence: the
    // first writer warp issues them after the planner kernel (below)
    if (STAGE && (!g.dev_planned || g.plan_ready)) row_prologue_k<STAGE>(smem, c, g, rl, bar);
  }
  __syncthreads();  // mbarriers initialised before anyone waits on them
  if (warp < P) {
    int j = warp;
    int tile = blockIdx.x + j * gridDim.x;
    // row inputs (axis values, libm log2) are plan-independent: the first
    // tile's staircase and W table overlap the planner kernel
    RowIn<NB> rin = load_row_in<NB, RB>(g, rl, min(tile, rl.tiles - 1), t.NW, lane);
    mbar_wait(bar, 0);
    for (; tile < rl.tiles; j += P, tile += P * gridDim.x) {
      const int slot = j % S, use = j / S;
      const RowIn<NB> cur = rin;
      {
        const int nt = tile + P * gridDim.x;
        if (nt < rl.tiles) rin = load_row_in<NB, RB>(g, rl, nt, t.NW, lane);
      }
      if (use > 0) mbar_wait(empty + slot, (use - 1) & 1);
#ifdef PM2L_TIMING
      if (lane == 0 && tile < 16384) rl.dbg_row[tile * 8] = t_entry;
#endif
      ROW_MARK(tile, 1);
      const bool first = j < P;
      build_tile<NB, STAGE, SEGW, RB>(c, g, rl, tile_xy(rl, tile, c.nK), cur,
                                  smem + rl.off_warp + slot * rl.warp_bytes, lane, tile,
                                  /*with_w=*/j >= nhelp,
                                  j < nhelp && !RB ? sready + j : nullptr,
                                  first ? bar + 1 : nullptr, first && g.dev_planned);
      __syncwarp();
      ROW_MARK(tile, 2);
      mbar_arrive(full + slot);
    }
  } else {
    const int cw = warp - P;
    if (cw < nhelp) {
      // W table of builder cw's first tile (position cw, slot cw)
      const int tile0 = blockIdx.x + cw * gridDim.x;
      uint8_t* wb0 = smem + rl.off_warp + cw * rl.warp_bytes;
      RowIn<NB> r0;
      if (tile0 < rl.tiles) r0 = load_row_in<NB, RB>(g, rl, tile0, t.NW, lane);
      mbar_wait(bar, 0);
      if (tile0 < rl.tiles && !RB)
        build_w_table<NB, STAGE>(c, g, r0, reinterpret_cast<double*>(wb0 + rl.w_W), lane);
      if (g.dev_planned) {
        pdl_wait();  // the planner kernel's per-k tables are complete and visible
        if (STAGE && cw == 0 && lane == 0 && !g.plan_ready) row_prologue_k<STAGE>(smem, c, g, rl, bar);
      }
      if (tile0 < rl.tiles && !RB) {
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
      rl.dbg_pdl[blockIdx.x * 4] = t_entry;
      rl.dbg_pdl[blockIdx.x * 4 + 1] = clock64();
    }
#endif
    pdl_wait();  // base table complete and visible
#ifdef PM2L_TIMING
    if (cw == 0 && lane == 0 && blockIdx.x < 4096) rl.dbg_pdl[blockIdx.x * 4 + 2] = clock64();
#endif
    for (int j = 0, tile = blockIdx.x; tile < rl.tiles; ++j, tile += gridDim.x) {
      const int slot = j % S, use = j / S;
      mbar_wait(full + slot, use & 1);
      if (j < nhelp) mbar_wait(wready + j, 0);
#ifdef PM2L_TIMING
      if (j == 0 && cw == 0 && lane == 0 && blockIdx.x < 4096) rl.dbg_pdl[blockIdx.x * 4 + 3] = clock64();
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

template <int NB, bool STAGE, int SEGW>
cudaError_t launch_rows_k(const TablesDev& t, const GridDev& g, const RowLaunch& rl,
                          const double* base, const LaunchOut& out, cudaStream_t s) {
  auto* fn = rl.rowblock ? grid_ring_kernel<NB, STAGE, SEGW, true, true>
             : rl.pair     ? grid_ring_kernel<NB, STAGE, SEGW, true, false>
                           : grid_ring_kernel<NB, STAGE, SEGW, false, false>;
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

}  // namespace gk
}  // namespace pm2l
