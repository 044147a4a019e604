// Device planner: the per-slice work of the host planner (tables.cpp
// build_grid) as one sm_100a kernel, so that a sweep's per-grid planning is
// GPU work in the same stream as the prediction (no host round trip, CUDA
// graph capturable).  For canonical axes (GridSpec: strictly ascending,
// values in [1, lut_n)) it writes exactly the GridDev arrays build_grid
// writes (tests compare them), plus the per-(curve, k) base table.
//
// plan_kernel roles, by block index:
//   [0, nkc)            one k chunk (kKChunk values) each: libm log2 from the
//                       per-device table, k-group insertion point, the k-only
//                       half of the one-class argmin (mn(k), gB(k)), the
//                       stable descending rank of mn inside the chunk
//                       (bitonic sort of (mn, index) in shared memory) and the
//                       per-group right cuts (kright)
//   nkc                 exact-record join (_kernels.pyx:107-110): every exact
//                       record whose (b, m, n, k) lies on the slice becomes a
//                       fix-up, bucketed by (m, n) row (counting sort)
//   nkc + 1             m / n logs, per-(value, wave class) tile counts, the
//                       unresolved-point statistics reset
//   nkc + 2 ...         base(c, k) = ref_dur*(k/ref_dim)*(ref_thr/thr(c, k))
//                       (compute.py:109-138), one (curve, 1024 k) block each
// Every comparison and FP64 operation is the host planner's, on the same
// bits (IEEE subtraction, |.| as ordered bits, lower_bound), so the plan is
// identical.  Violations of the canonical-axis contract set bits of
// GridDev::status instead of faulting.
#include <algorithm>

#include "common.cuh"

namespace pm2l {
namespace {

using namespace dev;

#ifndef PM2L_PLAN_THREADS
#define PM2L_PLAN_THREADS 512  // A/B: planner alone 12.2 -> 11.2 us, step 29.05 -> 28.9 us (128: slower, 1024: no better)
#endif
constexpr int kPlanThreads = PM2L_PLAN_THREADS;
constexpr int kBaseBlock = 1024;           // k values per base-table block
constexpr int kMaxBaseSamples = 256;       // samples staged per base block

__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;"); }

#ifdef PM2L_TIMING
#define PLAN_MARK(a, slot)                                                   \
  do {                                                                       \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                             \
      unsigned long long t_;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      (a).dbg[8 * blockIdx.x + (slot)] = t_;                                 \
    }                                                                        \
  } while (0)
#else
#define PLAN_MARK(a, slot) do {} while (0)
#endif

__device__ __forceinline__ void flag(uint32_t* status, uint32_t bit) {
  if (status) atomicOr(status, bit);
}

// index of v in the ascending array a[0..n), or -1
__device__ __forceinline__ int64_t find_sorted(const uint64_t* a, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return (lo < n && a[lo] == v) ? lo : -1;
}

struct PlanArgs {
  int nkc;           // k chunks
  int kparts;        // rank CTAs per k chunk
  int ranks;         // k ranks / kright needed (lookup kernel's byte maps)
  int nrec;          // record CTAs
  int nrow;          // row-range CTAs
  int kblocks;       // base-table k blocks per curve
  int stage_axes;    // record / row CTAs stage the axes in shared memory
  int stage_keys;    // row CTAs stage the records' (m, n) keys
  const double* lut;
  int64_t lut_n;
  double* base;
  unsigned long long* stats;
#ifdef PM2L_TIMING
  unsigned long long* dbg;  // diagnostic build: per-CTA globaltimer at entry / exit
#endif
};

// ----------------------------------------------------------------- k ranks
// One chunk of kKChunk k values is served by several CTAs; each computes the
// k-only quantities of the whole chunk in shared memory (a few dependent
// loads per k) and the rank of its own kRankPerCta k values by counting:
// rank(i) = #{j : mn_j > mn_i} + #{j < i : mn_j == mn_i}, the position in the
// stable descending order of mn (std::stable_sort in the host planner).  A
// warp counts for kRankPerWarp values at a time over lane-strided j.
#ifndef PM2L_RANK_PER_WARP
#define PM2L_RANK_PER_WARP 1  // measured: 1 (125 rank CTAs for C2) > 2 > 4 > 8
#endif
constexpr int kRankPerWarp = PM2L_RANK_PER_WARP;
constexpr int kRankPerCta = kRankPerWarp * (kPlanThreads / 32);

__device__ void plan_k_rank(const TablesDev& t, const GridDev& g, const PlanArgs& a, int chunk,
                            int part, uint8_t* smem) {
  const int64_t k0 = int64_t(chunk) * kKChunk;
  const int kc = int(::min((int64_t)kKChunk, g.nK - k0));
  uint64_t* mn_s = reinterpret_cast<uint64_t*>(smem);                 // [kKChunk]
  double* glk = reinterpret_cast<double*>(mn_s + kKChunk);            // [256]
  uint8_t* st_s = reinterpret_cast<uint8_t*>(glk + 256);              // [kKChunk]
  uint8_t* gb_s = st_s + kKChunk;                                     // [kKChunk]
  const int G = t.G, tid = threadIdx.x;
  constexpr int kPer = kKChunk / kPlanThreads;
  uint64_t kv[kPer];
#pragma unroll
  for (int h = 0; h < kPer; ++h) {
    const int i = tid + h * kPlanThreads;
    kv[h] = i < kc ? g.K[k0 + i] : 0;
  }
  for (int i = tid; i < G; i += kPlanThreads) glk[i] = t.grp_lk[i];
  __syncthreads();
  PLAN_MARK(a, 1);
  auto dk = [&](int gg, double qk) { return abs_bits(__dsub_rn(glk[gg], qk)); };
  double qv[kPer];  // every log2 gather in flight at once
#pragma unroll
  for (int h = 0; h < kPer; ++h) {
    const uint64_t k = kv[h];
    qv[h] = (k >= 1 && int64_t(k) < a.lut_n) ? __ldg(a.lut + k) : 0.0;
  }
#pragma unroll
  for (int h = 0; h < kPer; ++h) {
    const int i = tid + h * kPlanThreads;
    if (i >= kc) continue;
    const uint64_t k = kv[h];
    const bool ok = k >= 1 && int64_t(k) < a.lut_n;
    const double qk = qv[h];
    // #groups with grp_lk < qk (std::lower_bound)
    int lo = 0, hi = G;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (glk[mid] < qk) lo = mid + 1; else hi = mid;
    }
    const int start = lo;
    const uint64_t dkL = start > 0 ? dk(start - 1, qk) : ~0ull;
    const uint64_t dkR = start < G ? dk(start, qk) : ~0ull;
    const uint64_t mn = dkL < dkR ? dkL : dkR;
    int gb = start;
    if (start > 0 && dkL == mn) {
      gb = start - 1;
      while (gb > 0 && dk(gb - 1, qk) == mn) --gb;
    }
    mn_s[i] = mn;
    st_s[i] = uint8_t(start);
    gb_s[i] = uint8_t(gb);
    if (part == 0) {  // one CTA per chunk writes the per-k arrays and checks the axis
      const int64_t ik = k0 + i;
      const_cast<KInfo*>(g.kinfo)[ik] = KInfo{qk, start, 0};
      const_cast<double*>(g.logK)[ik] = qk;
      if (!ok || k >= (uint64_t(1) << 62)) flag(g.status, kPlanBadValue);
      if (ik > 0 && !(g.K[ik - 1] < k)) flag(g.status, kPlanUnsorted);
    }
  }
  if (!a.ranks) return;  // kinfo / logK only (direct resolve, sweep kernel)
  __syncthreads();
  PLAN_MARK(a, 2);
  const int lane = tid & 31, warp = tid >> 5;
  const int i0 = part * kRankPerCta + warp * kRankPerWarp;
  uint64_t mi[kRankPerWarp];
  int cnt[kRankPerWarp];
#pragma unroll
  for (int u = 0; u < kRankPerWarp; ++u) {
    mi[u] = i0 + u < kc ? mn_s[i0 + u] : 0;
    cnt[u] = 0;
  }
  if (i0 < kc) {
#pragma unroll 4
    for (int j = lane; j < kc; j += 32) {
      const uint64_t mj = mn_s[j];
#pragma unroll
      for (int u = 0; u < kRankPerWarp; ++u)
        cnt[u] += (mj > mi[u] || (mj == mi[u] && j < i0 + u)) ? 1 : 0;
    }
#pragma unroll
    for (int u = 0; u < kRankPerWarp; ++u)
      for (int o = 16; o; o >>= 1) cnt[u] += __shfl_xor_sync(0xFFFFFFFFu, cnt[u], o);
    if (lane < kRankPerWarp) {
      int r = 0;
#pragma unroll
      for (int u = 0; u < kRankPerWarp; ++u) r = lane == u ? cnt[u] : r;
      const int i = i0 + lane;
      if (i < kc) {
        const_cast<uint64_t*>(g.mn_sorted)[k0 + r] = mn_s[i];
        const_cast<uint32_t*>(g.kfast)[k0 + i] =
            uint32_t(r) | (uint32_t(gb_s[i]) << 16) | (uint32_t(st_s[i]) << 24);
      }
    }
  }
  // kright[chunk][g]: first chunk-local index whose insertion point exceeds
  // g (start is non-decreasing along an ascending k axis)
  if (part == 0) {
    int32_t* kright = const_cast<int32_t*>(g.kright);
    for (int gg = tid; gg < G; gg += kPlanThreads) {
      int l = 0, h = kc;
      while (l < h) {
        const int mid = (l + h) >> 1;
        if (st_s[mid] <= gg) l = mid + 1; else h = mid;
      }
      kright[int64_t(chunk) * G + gg] = l;
    }
  }
}

// ------------------------------------------------------- exact-record join
// Records are the tables' unique exact shapes sorted by (m, n, b, k), so one
// (m, n) row owns a contiguous range of them.  Record CTAs locate each
// record on the slice (fix-up entry, or ib = -1 when it is off the slice);
// row CTAs find each row's range.  Both are independent of each other.
__device__ void stage_axes(const GridDev& g, const PlanArgs& a, uint64_t* ax,
                           const uint64_t** Bs, const uint64_t** Ms, const uint64_t** Ns,
                           const uint64_t** Ks, bool with_bk) {
  const int64_t nbs = g.b_hi - g.b_lo;
  *Bs = g.B + g.b_lo; *Ms = g.M; *Ns = g.N; *Ks = g.K;
  if (!a.stage_axes) return;
  uint64_t* p = ax;
  for (int64_t i = threadIdx.x; i < g.nM; i += blockDim.x) p[i] = g.M[i];
  *Ms = p; p += g.nM;
  for (int64_t i = threadIdx.x; i < g.nN; i += blockDim.x) p[i] = g.N[i];
  *Ns = p; p += g.nN;
  if (!with_bk) return;
  for (int64_t i = threadIdx.x; i < nbs; i += blockDim.x) p[i] = g.B[g.b_lo + i];
  *Bs = p; p += nbs;
  for (int64_t i = threadIdx.x; i < g.nK; i += blockDim.x) p[i] = g.K[i];
  *Ks = p;
}

__device__ void plan_records(const TablesDev& t, const GridDev& g, const PlanArgs& a, int blk,
                             uint8_t* smem) {
  const int r = blk * kPlanThreads + threadIdx.x;
  const bool mine = r < t.n_mn;
  uint64_t c4[4] = {0, 0, 0, 0};
  if (mine)
    for (int j = 0; j < 4; ++j) c4[j] = t.ex_mn_coord[4 * int64_t(r) + j];
  const uint64_t *Bs, *Ms, *Ns, *Ks;
  stage_axes(g, a, reinterpret_cast<uint64_t*>(smem), &Bs, &Ms, &Ns, &Ks, true);
  __syncthreads();
  if (!mine) return;
  const int64_t ib = find_sorted(Bs, g.b_hi - g.b_lo, c4[0]);
  const int64_t im = ib < 0 ? -1 : find_sorted(Ms, g.nM, c4[1]);
  const int64_t jn = im < 0 ? -1 : find_sorted(Ns, g.nN, c4[2]);
  const int64_t ik = jn < 0 ? -1 : find_sorted(Ks, g.nK, c4[3]);
  const bool on = ik >= 0;
  const int32_t ci = t.ex_mn_curve[r];
  const_cast<FixEntry*>(g.fixr)[r] =
      FixEntry{on ? int32_t(ik) : -1, on ? int32_t(ib) : -1, ci, ci >= 0 ? t.wc_of[ci] : -1};
  const_cast<int64_t*>(g.fix_pos)[r] = on ? ((ib * g.nM + im) * g.nN + jn) * g.nK + ik : -1;
}

__device__ void plan_rows_rng(const TablesDev& t, const GridDev& g, const PlanArgs& a, int blk,
                              uint8_t* smem) {
  const uint64_t *Bs, *Ms, *Ns, *Ks;
  stage_axes(g, a, reinterpret_cast<uint64_t*>(smem), &Bs, &Ms, &Ns, &Ks, false);
  // the records' (m, n) keys, for the range searches
  uint64_t* km = reinterpret_cast<uint64_t*>(smem) + (a.stage_axes ? g.nM + g.nN : 0);
  const int R = t.n_mn;
  const bool stage_keys = a.stage_keys != 0;
  if (stage_keys)
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      km[2 * i] = t.ex_mn_coord[4 * int64_t(i) + 1];
      km[2 * i + 1] = t.ex_mn_coord[4 * int64_t(i) + 2];
    }
  __syncthreads();
  const int64_t row = int64_t(blk) * kPlanThreads + threadIdx.x;
  if (row >= g.nM * g.nN) return;
  const int64_t im = row / g.nN, jn = row - im * g.nN;
  const uint64_t m = Ms[im], n = Ns[jn];
  auto key_less = [&](int i, uint64_t qm, uint64_t qn, bool upper) {
    const uint64_t rm = stage_keys ? km[2 * i] : t.ex_mn_coord[4 * int64_t(i) + 1];
    const uint64_t rn = stage_keys ? km[2 * i + 1] : t.ex_mn_coord[4 * int64_t(i) + 2];
    return upper ? (rm < qm || (rm == qm && rn <= qn)) : (rm < qm || (rm == qm && rn < qn));
  };
  int lo = 0, hi = R;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (key_less(mid, m, n, false)) lo = mid + 1; else hi = mid;
  }
  int lo2 = lo, hi2 = R;
  while (lo2 < hi2) {
    const int mid = (lo2 + hi2) >> 1;
    if (key_less(mid, m, n, true)) lo2 = mid + 1; else hi2 = mid;
  }
  const_cast<int2*>(g.fixr_rng)[row] = make_int2(lo, lo2);
}

// ---------------------------------------------------- m / n axes, W inputs
__device__ void plan_mn(const TablesDev& t, const GridDev& g, const PlanArgs& a) {
  if (threadIdx.x == 0 && a.stats) {
    a.stats[0] = ~0ull;
    a.stats[1] = 0ull;
    a.stats[2] = 0ull;
  }
  for (int64_t i = threadIdx.x; i < g.nB; i += blockDim.x) {
    const uint64_t v = g.B[i];
    if (v == 0) flag(g.status, kPlanBadValue);
    if (i > 0 && !(g.B[i - 1] < v)) flag(g.status, kPlanUnsorted);
  }
  for (int ax = 0; ax < 2; ++ax) {
    const uint64_t* V = ax == 0 ? g.M : g.N;
    double* L = const_cast<double*>(ax == 0 ? g.logM : g.logN);
    const int64_t n = ax == 0 ? g.nM : g.nN;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t v = V[i];
      if (v == 0 || int64_t(v) >= a.lut_n || v >= (uint64_t(1) << 62)) flag(g.status, kPlanBadValue);
      if (i > 0 && !(V[i - 1] < v)) flag(g.status, kPlanUnsorted);
      L[i] = (v >= 1 && int64_t(v) < a.lut_n) ? a.lut[v] : 0.0;
    }
  }
}

// -------------------------------------------------------------- base table
__device__ void plan_base(const TablesDev& t, const GridDev& g, const PlanArgs& a, int blk) {
  __shared__ double sd[kMaxBaseSamples], sy[kMaxBaseSamples];
  const int c = blk / a.kblocks, kb = blk - c * a.kblocks;
  const int64_t k_lo = int64_t(kb) * kBaseBlock, k_hi = ::min((int64_t)g.nK, k_lo + kBaseBlock);
  const int lo = t.s_off[c], hi = t.s_off[c + 1], ns = hi - lo;
  double* base = a.base + int64_t(c) * g.nK;
  if (ns <= 0) {
    for (int64_t ik = k_lo + threadIdx.x; ik < k_hi; ik += blockDim.x) base[ik] = 0.0;
    return;
  }
  const bool staged = ns <= kMaxBaseSamples;
  if (staged)
    for (int j = threadIdx.x; j < ns; j += blockDim.x) {
      sd[j] = t.s_dims[lo + j];
      sy[j] = t.s_thrs[lo + j];
    }
  __syncthreads();
  for (int64_t ik = k_lo + threadIdx.x; ik < k_hi; ik += blockDim.x) {
    const double nd = __ull2double_rn(g.K[ik]);
    const double thr = staged ? interp_samples(sd, sy, 0, ns, nd)
                              : interp_samples(t.s_dims, t.s_thrs, lo, hi, nd);
    base[ik] = base_from_thr(t, c, nd, thr);
  }
}

// PM2L_PLAN_MINB (build macro, tuning): blocks per SM the register budget
// must allow; unset, the compiler picks (58 registers at 512 threads)
#ifdef PM2L_PLAN_MINB
#define PLAN_BOUNDS __launch_bounds__(kPlanThreads, PM2L_PLAN_MINB)
#else
#define PLAN_BOUNDS __launch_bounds__(kPlanThreads)
#endif
__global__ void PLAN_BOUNDS plan_kernel(TablesDev t, GridDev g, PlanArgs a) {
  pdl_release();  // the grid kernel may launch and run its table prologue now
  extern __shared__ __align__(16) uint8_t smem[];
  const int b = blockIdx.x;
#ifdef PM2L_TIMING
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
  const int nk = a.nkc * a.kparts;
  if (b < nk) plan_k_rank(t, g, a, b / a.kparts, b % a.kparts, smem);
  else if (b < nk + a.nrec) plan_records(t, g, a, b - nk, smem);
  else if (b < nk + a.nrec + a.nrow) plan_rows_rng(t, g, a, b - nk - a.nrec, smem);
  else if (b == nk + a.nrec + a.nrow) plan_mn(t, g, a);
  else plan_base(t, g, a, b - nk - a.nrec - a.nrow - 1);
#ifdef PM2L_TIMING
  __syncthreads();
  if (threadIdx.x == 0 && b < 1024) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    a.dbg[8 * b] = t0;
    a.dbg[8 * b + 7] = t1;
  }
#endif
}

// Plan buffer layout (256-byte aligned sections).
struct Layout {
  int64_t B, M, N, K, logM, logN, logK, kinfo, kfast, mn_sorted, kright, fix_pos, fixr,
      fixr_rng, status, total;
};

Layout layout(const TablesDev& t, const DPlanCaps& c) {
  Layout L{};
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = (o + std::max<int64_t>(bytes, 16) + 255) & ~int64_t(255);
    return at;
  };
  const int64_t nkc = (c.nK + kKChunk - 1) / kKChunk, R = t.n_mn;
  L.B = take(8 * c.nB); L.M = take(8 * c.nM); L.N = take(8 * c.nN); L.K = take(8 * c.nK);
  L.logM = take(8 * c.nM); L.logN = take(8 * c.nN); L.logK = take(8 * c.nK);
  L.kinfo = take(int64_t(sizeof(KInfo)) * c.nK);
  L.kfast = take(4 * c.nK); L.mn_sorted = take(8 * c.nK); L.kright = take(4 * nkc * t.G);
  L.fix_pos = take(8 * R);
  L.fixr = take(int64_t(sizeof(FixEntry)) * R);
  L.fixr_rng = take(8 * c.nM * c.nN);
  L.status = take(4);
  L.total = o + 256;
  return L;
}

constexpr int64_t kStageAxesBytes = 64 * 1024;
constexpr int64_t kStageKeysBytes = 48 * 1024;

}  // namespace

#ifdef PM2L_TIMING
unsigned long long*& plan_timing_buffer() {
  static unsigned long long* p = nullptr;
  return p;
}
#endif

bool dplan_supported(const TablesDev& t, const DPlanCaps& c) {
  // G < 256 and k chunks of kKChunk: the kfast packing; rows and axes fit
  // 31-bit launch indices
  return t.G >= 0 && t.G <= 255 && c.nK >= 1 && c.nK <= 65535 && c.nM >= 1 && c.nN >= 1 &&
         c.nB >= 1 && c.nM * c.nN <= (int64_t(1) << 30) && c.nB <= (int64_t(1) << 30);
}

int64_t dplan_bytes(const TablesDev& t, const DPlanCaps& c) { return layout(t, c).total; }

uint64_t* dplan_axis_slot(const TablesDev& t, const DPlanCaps& c, void* buf, int axis) {
  const Layout L = layout(t, c);
  const int64_t off[4] = {L.B, L.M, L.N, L.K};
  return reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(buf) + off[axis]);
}

GridDev dplan_grid(const TablesDev& t, const DPlanCaps& c, void* buf, const uint64_t* const axes[4],
                   const int64_t lens[4], int64_t b_lo, int64_t b_hi) {
  const Layout L = layout(t, c);
  uint8_t* p = static_cast<uint8_t*>(buf);
  GridDev g{};
  g.nB = lens[0]; g.nM = lens[1]; g.nN = lens[2]; g.nK = lens[3];
  g.b_lo = b_lo; g.b_hi = b_hi;
  const int64_t off[4] = {L.B, L.M, L.N, L.K};
  const uint64_t* ax[4];
  for (int a = 0; a < 4; ++a)
    ax[a] = axes && axes[a] ? axes[a] : reinterpret_cast<const uint64_t*>(p + off[a]);
  g.B = ax[0]; g.M = ax[1]; g.N = ax[2]; g.K = ax[3];
  g.logM = reinterpret_cast<const double*>(p + L.logM);
  g.logN = reinterpret_cast<const double*>(p + L.logN);
  g.logK = reinterpret_cast<const double*>(p + L.logK);
  g.kinfo = reinterpret_cast<KInfo*>(p + L.kinfo);
  g.kfast = reinterpret_cast<const uint32_t*>(p + L.kfast);
  g.mn_sorted = reinterpret_cast<const uint64_t*>(p + L.mn_sorted);
  g.kright = reinterpret_cast<const int32_t*>(p + L.kright);
  // one fix-up entry per unique exact record (ib == -1, fix_pos == -1 when
  // it is off the slice); coordinates and curves are the tables' own
  g.n_fix = t.n_mn;
  g.fix_pos = reinterpret_cast<const int64_t*>(p + L.fix_pos);
  g.fix_coord = t.ex_mn_coord;
  g.fix_curve = t.ex_mn_curve;
  g.fixr = reinterpret_cast<const FixEntry*>(p + L.fixr);
  g.fixr_rng = reinterpret_cast<const int2*>(p + L.fixr_rng);
  g.max_fix_row = t.n_mn;
  g.k_sorted = 1;  // canonical axes (a violation is reported in status)
  g.dev_planned = 1;
  g.status = reinterpret_cast<uint32_t*>(p + L.status);
  return g;
}

int launch_dplan(const TablesDev& t, const GridDev& g, double* base,
                 unsigned long long* nan_stats, bool ranks, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PlanArgs a{};
  a.nkc = int((g.nK + kKChunk - 1) / kKChunk);
  a.kparts = ranks ? int((std::min<int64_t>(g.nK, kKChunk) + kRankPerCta - 1) / kRankPerCta) : 1;
  a.ranks = ranks ? 1 : 0;
  a.nrec = (t.n_mn + kPlanThreads - 1) / kPlanThreads;
  a.nrow = int((g.nM * g.nN + kPlanThreads - 1) / kPlanThreads);
  a.kblocks = int((g.nK + kBaseBlock - 1) / kBaseBlock);
  a.lut = g.lut;
  a.lut_n = g.lut_n;
  a.base = base;
  a.stats = nan_stats;
#ifdef PM2L_TIMING
  static unsigned long long* dbg = nullptr;
  if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 8192);
  a.dbg = dbg;
  plan_timing_buffer() = dbg;
#endif
  const int64_t axes_bytes = 8 * ((g.b_hi - g.b_lo) + g.nM + g.nN + g.nK);
  a.stage_axes = axes_bytes <= kStageAxesBytes ? 1 : 0;
  a.stage_keys = 16ll * t.n_mn <= kStageKeysBytes ? 1 : 0;
  const int64_t rank_smem = 8 * kKChunk + 8 * 256 + 2 * kKChunk;
  const int64_t rec_smem = a.stage_axes ? axes_bytes : 0;
  const int64_t row_smem = (a.stage_axes ? 8 * (g.nM + g.nN) : 0) + (a.stage_keys ? 16ll * t.n_mn : 0);
  const int64_t smem = std::max(rank_smem, std::max(rec_smem, row_smem));
  const int blocks = a.nkc * a.kparts + a.nrec + a.nrow + 1 + t.C * a.kblocks;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return int(e);
  }
  // status bits are sticky until the owner reads them (pm2l_grid_dplan_status)
  plan_kernel<<<blocks, kPlanThreads, size_t(smem), s>>>(t, g, a);
  return int(cudaGetLastError());
}

}  // namespace pm2l
