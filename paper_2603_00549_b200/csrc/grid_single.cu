// Single-(m, n) grid kernel: the one-class nearest decision when every
// record of the triple sits at ONE (m, n) -- as in the attention / triton
// presets (row-block families: m = n = 1) -- for latency-only launches.
// No planner and no tile builds.
//
// Per (row, k), exactly nearest_one_class (grid.cu) with one distinct member:
//   dmin = D(m, n) = max(|lm - qm|, |ln - qn|) (every member's distance; the
//          first member in scan order wins the ties)
//   mn   = distance from qk to the nearest k-group, gB the leftmost such group
//   case A (mn <= dmin): the leftmost group within dmin of qk
//   case B:              gB
//   curve = cand_curve of that group's first member; base(curve, k) once
// and per batch value b: the exact record (b, m, n, k) if one exists
// (_kernels.pyx:107-110), else that curve; blocks / waves / rescale as
// common.cuh predict_point (compute.py:78-138).  Bit-identical to the other
// grid kernels (the same comparisons on the same bits).
//
// Work item = ((m, n) row, k), k fastest so a warp's stores for one batch
// value are contiguous; the item's resolve and base(curve, k) are done once
// and the thread walks a chunk of the slice's batch values (staged in shared
// memory), whose points are independent (unrolled for FP64 ILP).
#include <cstdint>

#include "grid_common.cuh"

namespace pm2l {
namespace gk {
namespace {

#ifndef SINGLE_MINB
#define SINGLE_MINB 3  // 80 registers (a few spilled): 3 CTAs per SM, measured 24.6 -> 22.5 us on C3
#endif
constexpr int kSingleThreads = 256;
constexpr int kSingleMaxRec = 64;
constexpr int kSingleMaxGroups = 1024;
constexpr int kSingleMaxB = 1024;   // batch values staged in shared memory
#ifndef SINGLE_UNROLL
#define SINGLE_UNROLL 8
#endif
constexpr int kSingleUnroll = SINGLE_UNROLL;  // batch values per work item, in flight together (FP64 ILP)
constexpr int kSingleMaxCurves = 32;
constexpr int kSingleMaxSamples = 512;

struct SingleLaunch {
  FastDiv d_item, d_nK, d_nN;   // work-item index decomposition (32-bit indices)
  int bchunk;                   // batch values per work item (launch_single)
#ifdef PM2L_TIMING
  unsigned long long* dbg;  // per CTA: entry, staged, first item resolved, exit (globaltimer)
#endif
};

#ifdef PM2L_TIMING
#define SINGLE_MARK(slot)                                                          \
  do {                                                                             \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                                   \
      unsigned long long t_;                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
      sl.dbg[4 * blockIdx.x + (slot)] = t_;                                        \
    }                                                                              \
  } while (0)
#else
#define SINGLE_MARK(slot) do {} while (0)
#endif

__device__ __forceinline__ int count_below_s(const double* v, int n, double q) {
  int pos = 0;
  for (int step = n > 0 ? 1 << (31 - __clz(n)) : 0; step > 0; step >>= 1)
    if (pos + step <= n && v[pos + step - 1] < q) pos += step;
  return pos;
}

// ceil(b * k / (tile_m * bpw)) of a row-block wave class through the
// combined divisor's magic when it fits (tables.cpp: slot 1), else the
// two-step ceil(ceil(b*k / tm) / bpw) -- the same integer
__device__ __forceinline__ uint64_t rb_waves(const WcParam& p, uint64_t bk) {
  if (p.tn && (p.ds[1] >> 16) && bk + p.tn - 1 <= 0xFFFFFFFFull) return ceil_div_p(p, 1, bk, p.tn);
  return ceil_div_p(p, 2, ceil_div_p(p, 0, bk, p.tm), p.bpw);
}

template <bool IDX32>
__global__ void __launch_bounds__(kSingleThreads, SINGLE_MINB) single_kernel(TablesDev t, GridDev g,
                                                                 SingleLaunch sl, LaunchOut out) {
  __shared__ double glk[kSingleMaxGroups];
  __shared__ int32_t gcur[kSingleMaxGroups];  // curve of each group's first member
  __shared__ uint64_t ex[4 * kSingleMaxRec];
  __shared__ int32_t exc[kSingleMaxRec];
  __shared__ uint64_t exk[kSingleMaxRec];     // distinct record k values, ascending
  __shared__ uint64_t bsm[kSingleMaxB];
  // the curves' samples and reference scalars (the per-item base(curve, k)
  // reads them from shared memory instead of a chain of dependent loads)
  __shared__ int32_t c_off[kSingleMaxCurves + 1];
  __shared__ double c_dims[kSingleMaxSamples], c_thrs[kSingleMaxSamples];
  __shared__ double c_ref[3 * kSingleMaxCurves];  // ref_dur, ref_dim, ref_thr
  __shared__ WcParam c_wp[kSingleMaxCurves];
  __shared__ uint8_t c_rb[kSingleMaxCurves];
  SINGLE_MARK(0);
  const int G = t.G, R = t.n_exact, C = t.C, S = t.n_samples, NXK = t.n_rec_k;
  const int64_t nb = g.b_hi - g.b_lo;
  const bool bstage = nb <= kSingleMaxB;
  // staging: every array's loads of one index issued together (one memory
  // round trip for the lot instead of one per array), then the stores
  {
    int n_max = G;
    n_max = max(n_max, 4 * R);
    n_max = max(n_max, S);
    n_max = max(n_max, C + 1);
    n_max = max(n_max, bstage ? int(nb) : 0);
    for (int i = threadIdx.x; i < n_max; i += blockDim.x) {
      const bool in_g = i < G, in_x = i < 4 * R, in_r = i < R, in_k = i < NXK, in_s = i < S,
                 in_c = i < C, in_o = i <= C, in_b = bstage && i < nb;
      const double v_glk = in_g ? t.grp_lk[i] : 0.0;
      const int32_t v_gc = in_g ? t.grp_curve0[i] : 0;
      const uint64_t v_ex = in_x ? t.ex_coord[i] : 0;
      const int32_t v_exc = in_r ? t.ex_curve[i] : 0;
      const uint64_t v_exk = in_k ? t.rec_k[i] : 0;
      const double v_sd = in_s ? t.s_dims[i] : 0.0, v_st = in_s ? t.s_thrs[i] : 0.0;
      const int32_t v_off = in_o ? t.s_off[i] : 0;
      const uint64_t v_b = in_b ? g.B[g.b_lo + i] : 0;
      double v_rd = 0.0, v_rm = 0.0, v_rt = 0.0;
      uint8_t v_rb = 0;
      WcParam v_wp{};
      if (in_c) {
        v_rd = t.ref_dur[i];
        v_rm = t.ref_dim[i];
        v_rt = t.ref_thr[i];
        v_rb = t.rowblock[i];
        v_wp = t.wcp_c[i];  // no dependent wc_of -> wcp load
      }
      if (in_g) { glk[i] = v_glk; gcur[i] = v_gc; }
      if (in_x) ex[i] = v_ex;
      if (in_r) exc[i] = v_exc;
      if (in_k) exk[i] = v_exk;
      if (in_s) { c_dims[i] = v_sd; c_thrs[i] = v_st; }
      if (in_o) c_off[i] = v_off;
      if (in_b) bsm[i] = v_b;
      if (in_c) {
        c_ref[3 * i] = v_rd;
        c_ref[3 * i + 1] = v_rm;
        c_ref[3 * i + 2] = v_rt;
        c_rb[i] = v_rb;
        c_wp[i] = v_wp;
      }
    }
  }
  __syncthreads();
  SINGLE_MARK(1);
  const double lm0 = t.cls_lm[0], ln0 = t.cls_ln[0];
  const int64_t nK = g.nK, nMN = g.nM * g.nN, plane = nMN * nK;
  const int64_t nbc = (nb + sl.bchunk - 1) / sl.bchunk;
  const int64_t per_bc = nMN * nK, work = per_bc * nbc;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  // base(c, k) = (ref_dur * (k / ref_dim)) * (ref_thr / thr(c, k)) from the
  // staged curve data (common.cuh base_from_thr / interp_samples)
  auto base_of_s = [&](int c, double nd) {
    const double thr = interp_samples(c_dims, c_thrs, c_off[c], c_off[c + 1], nd);
    return __dmul_rn(__dmul_rn(c_ref[3 * c], __ddiv_rn(nd, c_ref[3 * c + 1])),
                     __ddiv_rn(c_ref[3 * c + 2], thr));
  };
  // one work item (per lane); the loop below is warp-uniform so the warp
  // reconverges after every item (an exact-hit item's slower path would
  // otherwise leave the warp split for the rest of the loop)
  auto item = [&](int64_t w) {
    int64_t bc, row, ik, im, jn;
    if (IDX32) {  // magic divisions by the host-computed divisors
      const int wi = int(w);
      const int b_i = fdiv(wi, sl.d_item), rk = wi - b_i * int(per_bc);
      const int r_i = fdiv(rk, sl.d_nK), m_i = fdiv(r_i, sl.d_nN);
      bc = b_i;
      row = r_i;
      ik = rk - r_i * int(nK);
      im = m_i;
      jn = r_i - m_i * int(g.nN);
    } else {
      bc = w / per_bc;
      const int64_t rk = w - bc * per_bc;
      row = rk / nK;
      ik = rk - row * nK;
      im = row / g.nN;
      jn = row - im * g.nN;
    }
    const uint64_t m = g.M[im], n = g.N[jn], k = g.K[ik];
    double qm, qn, qk;
    if (g.dev_planned) {
      // device plans: host-libm log2 from the per-device table (the
      // contract: canonical axes with values in [1, lut_n))
      const bool ok = m >= 1 && n >= 1 && k >= 1 && m < uint64_t(g.lut_n) &&
                      n < uint64_t(g.lut_n) && k < uint64_t(g.lut_n);
      if (!ok) {
        if (g.status) atomicOr(g.status, uint32_t(kPlanBadValue));
        return;
      }
      qm = g.lut[m];
      qn = g.lut[n];
      qk = g.lut[k];
      if (g.status && bc == 0) {  // canonical-axis contract, as the planner checks it
        bool bad = ik > 0 && !(g.K[ik - 1] < k);
        if (ik == 0) bad |= (jn > 0 && !(g.N[jn - 1] < n)) || (jn == 0 && im > 0 && !(g.M[im - 1] < m));
        // the batch axis: its adjacent pairs spread over the items
        for (int64_t ib = w; ib + 1 < g.nB; ib += per_bc) bad |= !(g.B[ib] < g.B[ib + 1]);
        if (bad) atomicOr(g.status, uint32_t(kPlanUnsorted));
      }
    } else {
      qm = g.logM[im];
      qn = g.logN[jn];
      qk = g.logK[ik];
    }
    // row part: the members' (common) distance
    const uint64_t dmin = umax64(abs_bits(__dsub_rn(lm0, qm)), abs_bits(__dsub_rn(ln0, qn)));
    // k part
    const int start = count_below_s(glk, G, qk);
    auto dk = [&](int gg) { return abs_bits(__dsub_rn(glk[gg], qk)); };
    const uint64_t dkL = start > 0 ? dk(start - 1) : ~0ull;
    const uint64_t dkR = start < G ? dk(start) : ~0ull;
    const uint64_t mn = dkL < dkR ? dkL : dkR;
    int grp;
    if (mn <= dmin) {  // leftmost group within dmin
      if (dkL <= dmin) {
        grp = start - 1;
        while (grp > 0 && dk(grp - 1) <= dmin) --grp;
      } else {
        grp = start;
      }
    } else {           // leftmost nearest group
      if (dkL == mn) {
        grp = start - 1;
        while (grp > 0 && dk(grp - 1) == mn) --grp;
      } else {
        grp = start;
      }
    }
    const int ci = gcur[grp];
    const double nd = __ull2double_rn(k);
    // exact records on this (m, n, k): they can only sit on a recorded k
    int nhit = 0;
    uint64_t hb[4] = {0, 0, 0, 0};
    int32_t hc[4] = {0, 0, 0, 0};
    {
      int lo = 0;
      for (int step = NXK > 0 ? 1 << (31 - __clz(NXK)) : 0; step > 0; step >>= 1)
        if (lo + step <= NXK && exk[lo + step - 1] < k) lo += step;
      if (lo < NXK && exk[lo] == k)
        for (int r = 0; r < R; ++r)
          if (ex[4 * r + 3] == k && ex[4 * r + 1] == m && ex[4 * r + 2] == n) {
            const uint64_t rb_ = ex[4 * r];
            bool dup = false;  // a shape recorded twice: the first record wins
#pragma unroll
            for (int q = 0; q < 4; ++q) dup |= q < nhit && hb[q] == rb_;
            if (dup) continue;
#pragma unroll
            for (int q = 0; q < 4; ++q)  // constant indices: registers, not local memory
              if (q == nhit) {
                hb[q] = rb_;
                hc[q] = exc[r];
              }
            ++nhit;
          }
    }
    if (nhit > 4) nhit = -1;  // more than 4 batch values recorded here: scan per point
    const int64_t b0 = g.b_lo + bc * sl.bchunk;
    const int cnt = g.b_hi - b0 < sl.bchunk ? int(g.b_hi - b0) : sl.bchunk;
    double* o = out.lat + (bc * sl.bchunk * nMN + row) * nK + ik;
    if (w < int64_t(blockDim.x) * gridDim.x) SINGLE_MARK(2);
    // the item's curve, its base and wave parameters once
    double base = 0.0;
    WcParam prm{};
    bool rb = false;
    if (ci >= 0) {
      base = base_of_s(ci, nd);
      prm = c_wp[ci];
      rb = c_rb[ci] != 0;
    }
    const uint64_t* bv = bstage ? bsm + (b0 - g.b_lo) : g.B + b0;
    uint64_t rowc = 0;  // GEMM: ceil(m / tm) * ceil(n / tn) * split_k, per item
    if (ci >= 0 && !rb) rowc = ceil_div_p(prm, 0, m, prm.tm) * ceil_div_p(prm, 1, n, prm.tn) * prm.sk;
    // per batch value: the exact record's curve when (b, m, n, k) is recorded
    // (nhit > 0: the item's <= 4 recorded batch values; nhit < 0: a scan),
    // else the item's curve.  Points on the item's curve take the unrolled
    // arithmetic below; another curve (or none) the general path
    for (int j0 = 0; j0 < cnt; j0 += kSingleUnroll) {
#pragma unroll
      for (int jj = 0; jj < kSingleUnroll; ++jj) {
        const int j = j0 + jj;
        if (j >= cnt) continue;
        const uint64_t b = bv[j];
        int c = ci;
        if (nhit > 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nhit && hb[q] == b) c = hc[q];
        } else if (nhit < 0) {
          for (int r = 0; r < R; ++r)
            if (ex[4 * r] == b && ex[4 * r + 1] == m && ex[4 * r + 2] == n && ex[4 * r + 3] == k) {
              c = exc[r];
              break;
            }
        }
        double* oj = o + j * plane;
        if (c == ci && c >= 0) {
          const uint64_t wv = rb ? rb_waves(prm, b * k) : ceil_div_p(prm, 2, b * rowc, prm.bpw);
          const double wd = __ull2double_rn(wv);
          *oj = __dmul_rn(base, prm.rw == 1.0 ? wd : __ddiv_rn(wd, prm.rw));
        } else if (c < 0) {
          *oj = qnan();
          if (out.nan_stats) {
            atomicMin(out.nan_stats, (unsigned long long)(oj - out.lat));
            atomicAdd(out.nan_stats + 1, 1ull);
          }
        } else {
          const WcParam& p = c_wp[c];
          const double bs = base_of_s(c, nd);
          const uint64_t wv =
              c_rb[c] ? rb_waves(p, b * k)
                      : ceil_div_p(p, 2, b * ceil_div_p(p, 0, m, p.tm) * ceil_div_p(p, 1, n, p.tn) * p.sk,
                                   p.bpw);
          const double wd = __ull2double_rn(wv);
          *oj = __dmul_rn(bs, p.rw == 1.0 ? wd : __ddiv_rn(wd, p.rw));
        }
      }
    }
  };
  const int lane = threadIdx.x & 31;
  for (int64_t wb = blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31); wb < work; wb += stride) {
    if (wb + lane < work) item(wb + lane);
    __syncwarp();
  }
  __syncthreads();
  SINGLE_MARK(3);
}

__global__ void stats_reset_kernel(unsigned long long* stats) {
  stats[0] = ~0ull;
  stats[1] = 0;
  stats[2] = 0;
}

}  // namespace

bool single_ok(const TablesDev& t, const GridDev& g, const LaunchOut& out) {
  return !out.curve && t.single_mn && t.lowest_wins && t.G >= 1 && t.G <= kSingleMaxGroups &&
         t.n_exact <= kSingleMaxRec && t.R >= 1 && t.C <= kSingleMaxCurves &&
         t.n_samples <= kSingleMaxSamples &&
         (g.dev_planned ? g.lut != nullptr : (g.logM && g.logN && g.logK)) && g.nK > 0;
}

cudaError_t launch_single(const TablesDev& t, const GridDev& g, const LaunchOut& out, int stages,
                          cudaStream_t s) {
  if ((stages & kStageBase) && out.nan_stats) stats_reset_kernel<<<1, 1, 0, s>>>(out.nan_stats);
  if (stages & kStageGrid) {
    // persistent: one wave of resident CTAs (each stages the tables once)
    static int resident = 0;
    if (!resident) {
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, single_kernel<true>, kSingleThreads, 0) !=
              cudaSuccess || per_sm < 1)
        per_sm = 2;
      resident = per_sm;
    }
    // batch values per work item: one unrolled group (measured: larger
    // chunks, which share the item's resolve among more batch values, lose
    // more to the lower thread count than they save)
    const int64_t nb = g.b_hi - g.b_lo, rows = g.nM * g.nN * g.nK;
    const int bchunk = kSingleUnroll;
    const int64_t nbc = (nb + bchunk - 1) / bchunk;
    const int64_t work = rows * nbc;
    const int64_t want = (work + kSingleThreads - 1) / kSingleThreads;
    const int ctas = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sm_count()) * resident)));
    SingleLaunch sl{};
    sl.bchunk = bchunk;
#ifdef PM2L_TIMING
    sl.dbg = timing_buffers()[1];
#endif
    if (work < (int64_t(1) << 31)) {
      sl.d_item = fast_div_for(uint32_t(g.nM * g.nN * g.nK));
      sl.d_nK = fast_div_for(uint32_t(g.nK));
      sl.d_nN = fast_div_for(uint32_t(g.nN));
      single_kernel<true><<<ctas, kSingleThreads, 0, s>>>(t, g, sl, out);
    } else {
      single_kernel<false><<<ctas, kSingleThreads, 0, s>>>(t, g, sl, out);
    }
  }
  return cudaGetLastError();
}

}  // namespace gk
}  // namespace pm2l
