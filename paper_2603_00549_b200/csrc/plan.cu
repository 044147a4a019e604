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

constexpr int kPlanThreads = 1024;
constexpr int kBaseBlock = 1024;           // k values per base-table block
constexpr int kMaxBaseSamples = 256;       // samples staged per base block
constexpr int64_t kMaxJoinRows = 32768;    // (m, n) rows of a device-planned slice
constexpr int kMaxJoinRecords = 1 << 16;
constexpr int64_t kJoinStageBytes = 96 * 1024;

__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;"); }

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
  int kblocks;       // base-table k blocks per curve
  int stage_axes;    // join stages the axes in shared memory
  const double* lut;
  int64_t lut_n;
  double* base;
  unsigned long long* stats;
};

// ---------------------------------------------------------------- k chunk
__device__ void plan_k_chunk(const TablesDev& t, const GridDev& g, const PlanArgs& a, int chunk,
                             uint8_t* smem) {
  const int64_t k0 = int64_t(chunk) * kKChunk;
  const int kc = int(::min((int64_t)kKChunk, g.nK - k0));
  int P = 1;
  while (P < kc) P <<= 1;
  uint64_t* mn_s = reinterpret_cast<uint64_t*>(smem);                 // [kKChunk]
  double* glk = reinterpret_cast<double*>(mn_s + kKChunk);            // [256]
  uint16_t* idx_s = reinterpret_cast<uint16_t*>(glk + 256);           // [kKChunk]
  uint8_t* st_s = reinterpret_cast<uint8_t*>(idx_s + kKChunk);        // [kKChunk]
  uint8_t* gb_s = st_s + kKChunk;                                     // [kKChunk]
  const int G = t.G;
  for (int i = threadIdx.x; i < G; i += blockDim.x) glk[i] = t.grp_lk[i];
  __syncthreads();
  auto dk = [&](int gg, double qk) { return abs_bits(__dsub_rn(glk[gg], qk)); };
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (i >= kc) {
      mn_s[i] = 0;
      idx_s[i] = 0xFFFF;  // after every real entry (equal mn: larger index)
      continue;
    }
    const int64_t ik = k0 + i;
    const uint64_t k = g.K[ik];
    if (k == 0 || int64_t(k) >= a.lut_n || k >= (uint64_t(1) << 62)) flag(g.status, kPlanBadValue);
    if (ik > 0 && !(g.K[ik - 1] < k)) flag(g.status, kPlanUnsorted);
    const double qk = (k >= 1 && int64_t(k) < a.lut_n) ? a.lut[k] : 0.0;
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
    const_cast<KInfo*>(g.kinfo)[ik] = KInfo{qk, start, 0};
    const_cast<double*>(g.logK)[ik] = qk;
    mn_s[i] = mn;
    idx_s[i] = uint16_t(i);
    st_s[i] = uint8_t(start);
    gb_s[i] = uint8_t(gb);
  }
  __syncthreads();
  // bitonic sort, "a before b" = mn_a > mn_b || (mn_a == mn_b && idx_a < idx_b):
  // the stable descending order of mn (ties keep ascending k index)
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
        const int lo_i = 2 * i - (i & (stride - 1));
        const int hi_i = lo_i + stride;
        const bool up = (lo_i & size) == 0;  // this run ascends in "before" order
        const uint64_t ma = mn_s[lo_i], mb = mn_s[hi_i];
        const uint16_t ia = idx_s[lo_i], ib = idx_s[hi_i];
        const bool b_first = mb > ma || (mb == ma && ib < ia);
        if (b_first == up) {
          mn_s[lo_i] = mb; mn_s[hi_i] = ma;
          idx_s[lo_i] = ib; idx_s[hi_i] = ia;
        }
      }
      __syncthreads();
    }
  }
  uint32_t* kfast = const_cast<uint32_t*>(g.kfast);
  uint64_t* mn_sorted = const_cast<uint64_t*>(g.mn_sorted);
  for (int r = threadIdx.x; r < kc; r += blockDim.x) {
    const int i = idx_s[r];
    mn_sorted[k0 + r] = mn_s[r];
    kfast[k0 + i] = uint32_t(r) | (uint32_t(gb_s[i]) << 16) | (uint32_t(st_s[i]) << 24);
  }
  // kright[chunk][g]: first chunk-local index whose insertion point exceeds
  // g (start is non-decreasing along an ascending k axis)
  int32_t* kright = const_cast<int32_t*>(g.kright);
  for (int gg = threadIdx.x; gg < G; gg += blockDim.x) {
    int l = 0, h = kc;
    while (l < h) {
      const int mid = (l + h) >> 1;
      if (st_s[mid] <= gg) l = mid + 1; else h = mid;
    }
    kright[int64_t(chunk) * G + gg] = l;
  }
}

// ------------------------------------------------------- exact-record join
__device__ void plan_join(const TablesDev& t, const GridDev& g, const PlanArgs& a,
                          uint8_t* smem) {
  const int64_t nbs = g.b_hi - g.b_lo, rows = g.nM * g.nN;
  int32_t* cnt = reinterpret_cast<int32_t*>(smem);  // [rows + 1]
  uint64_t* ax = reinterpret_cast<uint64_t*>(smem + ((4 * (rows + 1) + 15) & ~int64_t(15)));
  const uint64_t* Bs = g.B + g.b_lo;
  const uint64_t* Ms = g.M;
  const uint64_t* Ns = g.N;
  const uint64_t* Ks = g.K;
  if (a.stage_axes) {
    uint64_t* p = ax;
    for (int64_t i = threadIdx.x; i < nbs; i += blockDim.x) p[i] = Bs[i];
    Bs = p; p += nbs;
    for (int64_t i = threadIdx.x; i < g.nM; i += blockDim.x) p[i] = Ms[i];
    Ms = p; p += g.nM;
    for (int64_t i = threadIdx.x; i < g.nN; i += blockDim.x) p[i] = Ns[i];
    Ns = p; p += g.nN;
    for (int64_t i = threadIdx.x; i < g.nK; i += blockDim.x) p[i] = Ks[i];
    Ks = p;
  }
  for (int64_t r = threadIdx.x; r <= rows; r += blockDim.x) cnt[r] = 0;
  __syncthreads();
  const int R = t.n_exact;
  struct Hit {
    int64_t ib, im, jn, ik;
  };
  auto locate = [&](int r) -> Hit {
    const uint64_t* c4 = t.ex_coord + 4 * int64_t(r);
    Hit h;
    h.ib = find_sorted(Bs, nbs, c4[0]);
    h.im = h.ib < 0 ? -1 : find_sorted(Ms, g.nM, c4[1]);
    h.jn = h.im < 0 ? -1 : find_sorted(Ns, g.nN, c4[2]);
    h.ik = h.jn < 0 ? -1 : find_sorted(Ks, g.nK, c4[3]);
    return h;
  };
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const Hit h = locate(r);
    if (h.ik >= 0) atomicAdd(&cnt[h.im * g.nN + h.jn], 1);
  }
  __syncthreads();
  // exclusive scan of the row counts -> fixr_off[0..rows] (one contiguous
  // segment per thread, then a block scan of the segment sums)
  __shared__ int32_t part[kPlanThreads];
  const int64_t n = rows + 1;
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t s0 = ::min((int64_t)n, threadIdx.x * per), s1 = ::min((int64_t)n, s0 + per);
  int32_t sum = 0;
  for (int64_t i = s0; i < s1; ++i) sum += cnt[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < int(blockDim.x); off <<= 1) {
    const int32_t v = threadIdx.x >= unsigned(off) ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = part[threadIdx.x] - sum;  // exclusive prefix of this segment
  int32_t* fixr_off = const_cast<int32_t*>(g.fixr_off);
  for (int64_t i = s0; i < s1; ++i) {
    const int32_t c = cnt[i];
    cnt[i] = run;  // becomes the scatter cursor
    fixr_off[i] = run;
    run += c;
  }
  if (threadIdx.x == blockDim.x - 1) *const_cast<int32_t*>(g.n_fix_dev) = part[blockDim.x - 1];
  __syncthreads();
  FixEntry* fixr = const_cast<FixEntry*>(g.fixr);
  int64_t* fix_pos = const_cast<int64_t*>(g.fix_pos);
  uint64_t* fix_coord = const_cast<uint64_t*>(g.fix_coord);
  int32_t* fix_curve = const_cast<int32_t*>(g.fix_curve);
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const Hit h = locate(r);
    if (h.ik < 0) continue;
    const int64_t row = h.im * g.nN + h.jn;
    const int slot = atomicAdd(&cnt[row], 1);
    const int32_t ci = t.ex_curve[r];
    fixr[slot] = FixEntry{int32_t(h.ik), int32_t(h.ib), ci, slot};
    fix_pos[slot] = ((h.ib * g.nM + h.im) * g.nN + h.jn) * g.nK + h.ik;
    const uint64_t* c4 = t.ex_coord + 4 * int64_t(r);
    for (int j = 0; j < 4; ++j) fix_coord[4 * int64_t(slot) + j] = c4[j];
    fix_curve[slot] = ci;
  }
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
  if (g.cm_tab) {
    // ceil(m / tile_m) and ceil(n / tile_n) * split_k per wave class, in u64
    // exactly like the host planner (and the reference's block product)
    uint64_t* cm = const_cast<uint64_t*>(g.cm_tab);
    uint64_t* cn = const_cast<uint64_t*>(g.cn_tab);
    const int NW = t.NW;
    for (int64_t e = threadIdx.x; e < g.nM * NW; e += blockDim.x) {
      const WcParam& p = t.wcp[e % NW];
      cm[e] = (g.M[e / NW] + p.tm - 1) / p.tm;
    }
    for (int64_t e = threadIdx.x; e < g.nN * NW; e += blockDim.x) {
      const WcParam& p = t.wcp[e % NW];
      cn[e] = ((g.N[e / NW] + p.tn - 1) / p.tn) * p.sk;
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

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(TablesDev t, GridDev g, PlanArgs a) {
  pdl_release();  // the grid kernel may launch and run its table prologue now
  extern __shared__ __align__(16) uint8_t smem[];
  const int b = blockIdx.x;
  if (b < a.nkc) plan_k_chunk(t, g, a, b, smem);
  else if (b == a.nkc) plan_join(t, g, a, smem);
  else if (b == a.nkc + 1) plan_mn(t, g, a);
  else plan_base(t, g, a, b - a.nkc - 2);
}

// Plan buffer layout (256-byte aligned sections).
struct Layout {
  int64_t B, M, N, K, logM, logN, logK, kinfo, kfast, mn_sorted, kright, cm, cn, fix_pos,
      fix_coord, fix_curve, fixr, fixr_off, n_fix, status, total;
};

Layout layout(const TablesDev& t, const DPlanCaps& c) {
  Layout L{};
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = (o + std::max<int64_t>(bytes, 16) + 255) & ~int64_t(255);
    return at;
  };
  const int64_t nkc = (c.nK + kKChunk - 1) / kKChunk, R = t.n_exact;
  L.B = take(8 * c.nB); L.M = take(8 * c.nM); L.N = take(8 * c.nN); L.K = take(8 * c.nK);
  L.logM = take(8 * c.nM); L.logN = take(8 * c.nN); L.logK = take(8 * c.nK);
  L.kinfo = take(int64_t(sizeof(KInfo)) * c.nK);
  L.kfast = take(4 * c.nK); L.mn_sorted = take(8 * c.nK); L.kright = take(4 * nkc * t.G);
  L.cm = take(8 * c.nM * t.NW); L.cn = take(8 * c.nN * t.NW);
  L.fix_pos = take(8 * R); L.fix_coord = take(32 * R); L.fix_curve = take(4 * R);
  L.fixr = take(int64_t(sizeof(FixEntry)) * R);
  L.fixr_off = take(4 * (c.nM * c.nN + 1));
  L.n_fix = take(4); L.status = take(4);
  L.total = o + 256;
  return L;
}

int64_t join_smem(const GridDev& g, bool stage) {
  const int64_t rows = g.nM * g.nN;
  int64_t s = (4 * (rows + 1) + 15) & ~int64_t(15);
  if (stage) s += 8 * ((g.b_hi - g.b_lo) + g.nM + g.nN + g.nK);
  return s;
}

}  // namespace

bool dplan_supported(const TablesDev& t, const DPlanCaps& c) {
  return t.G >= 0 && t.G <= 255 && c.nK >= 1 && c.nK <= 65535 && c.nM * c.nN + 1 <= kMaxJoinRows &&
         t.n_exact <= kMaxJoinRecords && c.nM >= 1 && c.nN >= 1 && c.nB >= 1;
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
  if (t.all_gemm && t.NW > 0) {
    g.cm_tab = reinterpret_cast<const uint64_t*>(p + L.cm);
    g.cn_tab = reinterpret_cast<const uint64_t*>(p + L.cn);
  }
  g.n_fix = t.n_exact;  // capacity; the planned count is n_fix_dev
  g.fix_pos = reinterpret_cast<const int64_t*>(p + L.fix_pos);
  g.fix_coord = reinterpret_cast<const uint64_t*>(p + L.fix_coord);
  g.fix_curve = reinterpret_cast<const int32_t*>(p + L.fix_curve);
  g.fixr_off = reinterpret_cast<const int32_t*>(p + L.fixr_off);
  g.fixr = reinterpret_cast<const FixEntry*>(p + L.fixr);
  g.max_fix_row = t.n_exact;
  g.k_sorted = 1;  // canonical axes (a violation is reported in status)
  g.dev_planned = 1;
  g.n_fix_dev = reinterpret_cast<const int32_t*>(p + L.n_fix);
  g.status = reinterpret_cast<uint32_t*>(p + L.status);
  return g;
}

int launch_dplan(const TablesDev& t, const GridDev& g, double* base,
                 unsigned long long* nan_stats, void* stream) {
  const double* lut = g.lut;
  const int64_t lut_n = g.lut_n;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PlanArgs a{};
  a.nkc = int((g.nK + kKChunk - 1) / kKChunk);
  a.kblocks = int((g.nK + kBaseBlock - 1) / kBaseBlock);
  a.lut = lut;
  a.lut_n = lut_n;
  a.base = base;
  a.stats = nan_stats;
  const int64_t chunk_smem = 8 * kKChunk + 8 * 256 + 2 * kKChunk + 2 * kKChunk;
  a.stage_axes = join_smem(g, true) <= kJoinStageBytes + 4 * (g.nM * g.nN + 1) ? 1 : 0;
  const int64_t smem = std::max(chunk_smem, join_smem(g, a.stage_axes != 0));
  const int blocks = a.nkc + 2 + t.C * a.kblocks;
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
