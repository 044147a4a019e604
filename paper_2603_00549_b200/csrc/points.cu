// Explicit-descriptor mode: n ops given as 16-byte {b, m, n, k} records.
//   points_kernel        ConfigResolver.resolve (pm2lat/compute.py:251-268):
//                        exact record first, else the nearest record by
//                        Chebyshev distance in log2 space (first scan index
//                        on ties), then the canonical prediction
//                        (compute.py:163-193)
//   points_curve_kernel  predict_generic with an explicit curve (no resolution)
//
// One op per lane.  The exact record comes from a hash whose slot tags sit in
// shared memory; for one-class tables (every shipped preset) the nearest
// search is the grid kernel's decision split into a k part (nearest k-group)
// and a member part over the row decomposition of the class (distinct log m
// rows x distinct log n columns, with each row's nearest present column per
// column insertion point precomputed: TablesDev::rw_lr); other tables take
// the k-group sweep over the member classes staged in shared memory.
#include <algorithm>

#include "common.cuh"

// PTS_VARIANT (diagnostic builds only, wrong results): 1 no nearest search,
// 2 no prediction tail, 3 no exact lookup, 4 no log2 loads, 5 = 1 + 2
#ifndef PTS_VARIANT
#define PTS_VARIANT 0
#endif
#ifndef PTS_MINB
#define PTS_MINB 4  // 64 registers: 4 CTAs per SM (measured best; 5 spills)
#endif
#ifndef PTS_PAIR
#define PTS_PAIR 1  // 2 measured slower (spills at 64 registers, no gain at 80)
#endif

namespace pm2l {
namespace {

using namespace dev;

constexpr int kTagSmemSlots = 4096;       // exact-hash tags staged in shared memory up to 16 KB
constexpr int kPointsPerLane = PTS_PAIR;  // one-class ops per lane per iteration (interleaved)

__device__ int exact_lookup(const TablesDev& t, uint64_t b, uint64_t m, uint64_t n, uint64_t k,
                            int* curve, int* record) {
  int lo = 0, hi = t.n_exact;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint64_t* e = t.ex_coord + 4 * mid;
    const bool eq = e[0] == b && e[1] == m && e[2] == n && e[3] == k;
    if (eq) {
      *curve = t.ex_curve[mid];
      *record = t.ex_rec[mid];
      return 1;
    }
    const bool less = e[0] != b ? e[0] < b : e[1] != m ? e[1] < m : e[2] != n ? e[2] < n : e[3] < k;
    if (less) lo = mid + 1; else hi = mid;
  }
  return 0;
}

struct PointSmem {
  const double* lm;
  const double* ln;
  const double* glk;
  const int32_t* gcls;
  const int32_t* gstart;
  const int32_t* cstart;
  const int32_t* csize;
  const int32_t* gidx;
};

__device__ __forceinline__ uint64_t member_d(const PointSmem& S, int j, double qm, double qn) {
  return umax64(abs_bits(__dsub_rn(S.lm[j], qm)), abs_bits(__dsub_rn(S.ln[j], qn)));
}

__device__ __forceinline__ uint64_t class_min(const PointSmem& S, int c, double qm, double qn) {
  uint64_t dmin = ~0ull;
  const int s = S.cstart[c], e = s + S.csize[c];
  for (int j = s; j < e; ++j) {
    const uint64_t d = member_d(S, j, qm, qn);
    dmin = d < dmin ? d : dmin;
  }
  return dmin;
}

// first member (scan order) of group g whose D <= best -> candidate scan index
__device__ __forceinline__ int first_within(const PointSmem& S, int g, uint64_t best, double qm,
                                            double qn) {
  const int c = S.gcls[g], s = S.cstart[c], e = s + S.csize[c];
  for (int j = s; j < e; ++j)
    if (member_d(S, j, qm, qn) <= best) return S.gidx[S.gstart[g] + (j - s)];
  return 0x7FFFFFFF;  // unreachable when best >= the class minimum
}

template <bool G32>
__device__ int nearest_point(const TablesDev& t, const PointSmem& S, double qm, double qn,
                             double qk, uint64_t* out_best) {
  // insertion point of qk among the ascending group lk values
  int lo = 0, hi = t.G;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (S.glk[mid] < qk) lo = mid + 1; else hi = mid;
  }
  uint64_t best = ~0ull;
  uint32_t mask = 0;
  int best_i = 0x7FFFFFFF;
  int cached = -1;
  uint64_t cached_min = 0;
  auto visit = [&](int g) -> bool {
    const uint64_t dk = abs_bits(__dsub_rn(S.glk[g], qk));
    if (dk > best) return false;
    const int c = S.gcls[g];
    if (c != cached) {
      cached = c;
      cached_min = class_min(S, c, qm, qn);
    }
    const uint64_t dg = umax64(dk, cached_min);
    if (G32) {
      if (dg < best) { best = dg; mask = 1u << g; }
      else if (dg == best) mask |= 1u << g;
    } else if (dg <= best) {
      const int idx = first_within(S, g, dg, qm, qn);
      if (dg < best || idx < best_i) best_i = idx;
      best = dg;
    }
    return true;
  };
  for (int g = lo; g < t.G; ++g)
    if (!visit(g)) break;
  for (int g = lo - 1; g >= 0; --g)
    if (!visit(g)) break;
  if (G32) {
    while (mask) {
      const int g = __ffs(mask) - 1;
      mask &= mask - 1;
      const int idx = first_within(S, g, best, qm, qn);
      best_i = idx < best_i ? idx : best_i;
    }
  }
  *out_best = best;
  return best_i;
}

// Exact record of a u32 descriptor through the hash (TablesDev::xh_*):
// linear probing over the slot tags (shared memory when they fit) from
// xh_hash until the key or an empty slot; the full key is read only on a
// tag match.
__device__ __forceinline__ int exact_hash(const TablesDev& t, const uint32_t* tags, uint4 s,
                                          int* curve, int* record) {
  uint32_t h = xh_hash(s.x, s.y, s.z, s.w) & uint32_t(t.xh_mask);
  const uint32_t tg = xh_tag(s.x, s.y, s.z, s.w);
  for (;;) {
    const uint32_t u = tags[h];
    if (u == 0) return 0;
    if (u == tg) {
      const uint4 k = __ldg(t.xh_key + h);
      if (k.x == s.x && k.y == s.y && k.z == s.z && k.w == s.w) {
        const int2 v = __ldg(t.xh_val + h);
        *curve = v.x;
        *record = v.y;
        return 1;
      }
    }
    h = (h + 1) & uint32_t(t.xh_mask);
  }
}

// host-libm log2 of a query coordinate: the per-device table below lut_n,
// else the caller's sorted extension; false when neither holds it
__device__ __forceinline__ bool query_log2(const LogSource& L, uint32_t x, double* out) {
  if (x < L.lut_n) {
    *out = __ldg(L.lut + x);
    return true;
  }
  int lo = 0, hi = int(L.n_ext);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(L.ext_coord + mid) < x) lo = mid + 1; else hi = mid;
  }
  if (lo < L.n_ext && __ldg(L.ext_coord + lo) == x) {
    *out = __ldg(L.ext_log + lo);
    return true;
  }
  return false;
}

struct QueryLogs {
  double m, n, k;
  bool ok;
};

// the three query logs of a descriptor (zero coordinates give ok = false
// with zeros: the op is invalid and its logs unused)
__device__ __forceinline__ QueryLogs query_logs(const LogSource& L, uint4 s) {
  QueryLogs q{0.0, 0.0, 0.0, false};
  if (s.y && s.z && s.w) {
    const bool a = query_log2(L, s.y, &q.m), b = query_log2(L, s.z, &q.n),
               c = query_log2(L, s.w, &q.k);
    q.ok = a && b && c;
  }
  return q;
}

__device__ __forceinline__ double dabs_sub(double a, double b) { return fabs(__dsub_rn(a, b)); }

// smallest power of two > n: sorted shared arrays padded with +inf to it
// take the unguarded search below
__host__ __device__ __forceinline__ int pow2_above(int n) {
  int p = 1;
  while (p <= n) p <<= 1;
  return p;
}

// number of v[0..np2) below q, v ascending and padded with +inf to np2 (a
// power of two > the real length): the same trip count in every lane and
// no bounds test per step
__device__ __forceinline__ int count_below_p2(const double* v, int np2, double q) {
  int pos = 0;
  for (int step = np2 >> 1; step > 0; step >>= 1) pos += v[pos + step - 1] < q ? step : 0;
  return pos;
}

struct RowSmem {
  const double* rlm;      // [NR] distinct member log m, ascending
  const double* cln;      // [NCl] distinct member log n, ascending
  const uint64_t* rmask;  // [NR] present columns of each row
  const uint64_t* cmask;  // [NCl] present rows of each column
  const int32_t* roff;    // [NR+1]
  const int32_t* rpos;    // [members] first position in the class member list
  const double2* lr;      // [NR x (NCl + 1)] nearest present column per side (TablesDev::rw_lr)
  int NR, NCl;
};

// The member part of the one-class decision from the row decomposition, with
// dm_i = |lm_i - qm| per row and dn_j = |ln_j - qn| per column (the member
// (i, j) has D = max(dm_i, dn_j)).  Rows and columns are ascending, so with
// pc the insertion point of qn every column distance is a difference of
// known sign (IEEE subtraction is exact in sign and monotone: |a - b| =
// b - a for a < b), V-shaped around pc:
//  * row pass (every row, a fixed trip count: no divergence): per row the
//    nearest present column is the highest present column below pc or the
//    lowest at or above it (TablesDev::rw_lr), so D_i = max(dm_i, nd_i) is
//    the row minimum; dmin = min_i D_i, irow = the first row attaining it
//    (strict <), and the rows within mn as a mask;
//  * column pass: the columns within dmin and within mn as masks;
//  * case A (mn <= dmin): the argmin is the first member with D <= dmin --
//    row irow (no earlier row reaches dmin), its lowest present column
//    within dmin;  case B: the first member with D <= mn -- the lowest row
//    within mn holding a present column within mn, that column.
// (Branch-free passes beat outward scans with early exits and lazy
// column searches here: measured, the divergence costs more than the
// rows it skips.)
// Returns the member's class position; *dmin_out = dmin.
template <class Mask, int P>  // Mask: uint32_t when rows and columns are <= 32, else uint64_t;
                              // P queries interleaved (independent FP64 chains per row)
__device__ __forceinline__ void member_rows(const RowSmem& W, const double* qm, const double* qn,
                                            const double* mn, double* dmin_out, int* pos_out) {
  constexpr int kBits = 8 * int(sizeof(Mask));
  const double INF = __longlong_as_double(0x7FF0000000000000ll);
  auto ffs = [](Mask x) { return kBits == 32 ? __ffs(uint32_t(x)) : __ffsll(static_cast<long long>(x)); };
  const int ld = W.NCl + 1, NClp = pow2_above(W.NCl);
  const double2* lr[P];
  double dmin[P];
  int irow[P];
  Mask rows_mn[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    lr[p] = W.lr + count_below_p2(W.cln, NClp, qn[p]);  // row i's neighbours of pc at lr[i * ld]
    dmin[p] = INF;
    irow[p] = 0;
    rows_mn[p] = 0;
  }
  for (int i = 0; i < W.NR; ++i) {  // fixed trip count: no divergence
    const double lmi = W.rlm[i];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const double dm = dabs_sub(lmi, qm[p]);
      // rw_lr holds -inf for an empty lower side and +inf for an empty upper one
      const double2 v = lr[p][i * ld];
      const double dl = __dsub_rn(qn[p], v.x), dr = __dsub_rn(v.y, qn[p]);
      const double nd = dl < dr ? dl : dr;
      const double D = dm > nd ? dm : nd;
      if (D < dmin[p]) {
        dmin[p] = D;
        irow[p] = i;
      }
      rows_mn[p] |= Mask(dm <= mn[p]) << i;
    }
  }
  Mask cols_d[P], cols_mn[P];
#pragma unroll
  for (int p = 0; p < P; ++p) cols_d[p] = cols_mn[p] = 0;
  for (int j = 0; j < W.NCl; ++j) {  // the columns within dmin and within mn
    const double lnj = W.cln[j];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const double dn = dabs_sub(lnj, qn[p]);
      cols_d[p] |= Mask(dn <= dmin[p]) << j;
      cols_mn[p] |= Mask(dn <= mn[p]) << j;
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    int i = irow[p];
    Mask cols = Mask(W.rmask[i]) & cols_d[p];
    if (!(mn[p] <= dmin[p])) {
      cols = 0;
      for (Mask rr = rows_mn[p]; rr && !cols; rr &= rr - 1) {
        i = ffs(rr) - 1;
        cols = Mask(W.rmask[i]) & cols_mn[p];
      }
    }
    const int j = ffs(cols) - 1;
    dmin_out[p] = dmin[p];
    const Mask before = (Mask(1) << j) - 1;
    const int rank = kBits == 32 ? __popc(uint32_t(Mask(W.rmask[i]) & before))
                                 : __popcll(static_cast<unsigned long long>(Mask(W.rmask[i]) & before));
    pos_out[p] = W.rpos[W.roff[i] + rank];
  }
}

// One member class (every shipped preset; equal logs imply equal
// coordinates): the grid kernel's nearest_one_class decision per op.  The
// k part: mn = distance from qk to the nearest k-group.  The member part:
// the row walk above when the class decomposes (ROWS), else one pass over
// the members -- dmin and its first member (case A: mn <= dmin) and the
// first member within mn (case B).  Returns the original candidate scan
// index; *out_best = the distance as ordered |double| bits.
template <int ROWS, int P>  // ROWS: 0 member pass, 1 rows (u32 masks), 2 rows (u64 masks);
                           // P queries (rows only) interleaved
__device__ void nearest_point_one_class(const TablesDev& t, const PointSmem& S, const RowSmem& W,
                                        const double* qm, const double* qn, const double* qk,
                                        int* out_rec, uint64_t* out_best) {
  const int G = t.G, Gp = pow2_above(G);
  int start[P];
  uint64_t dkL[P], mn[P];
  double mnd[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    start[p] = count_below_p2(S.glk, Gp, qk[p]);
    dkL[p] = start[p] > 0 ? abs_bits(__dsub_rn(S.glk[start[p] - 1], qk[p])) : ~0ull;
    const uint64_t dkR = start[p] < G ? abs_bits(__dsub_rn(S.glk[start[p]], qk[p])) : ~0ull;
    mn[p] = dkL[p] < dkR ? dkL[p] : dkR;
    // distances are non-negative finite doubles, so FP64 order is the order
    // of their |.| bits: compare them as doubles (DSETP)
    mnd[p] = __longlong_as_double(static_cast<long long>(mn[p]));
  }
  __syncwarp();  // every lane calls this (points_kernel): reconverge
  int pos[P];
  uint64_t dmin[P];
  if (ROWS) {
    double dm[P];
    if (ROWS == 1) member_rows<uint32_t, P>(W, qm, qn, mnd, dm, pos);
    else member_rows<uint64_t, P>(W, qm, qn, mnd, dm, pos);
#pragma unroll
    for (int p = 0; p < P; ++p) dmin[p] = abs_bits(dm[p]);
  } else {
    const int CM = S.csize[0];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double dminf = __longlong_as_double(0x7FF0000000000000ll);  // +inf
      int argmin = 0, first_mn = -1;
      for (int j = 0; j < CM; ++j) {
        const double d = fmax(fabs(__dsub_rn(S.lm[j], qm[p])), fabs(__dsub_rn(S.ln[j], qn[p])));
        if (d < dminf) { dminf = d; argmin = j; }
        if (first_mn < 0 && d <= mnd[p]) first_mn = j;
      }
      dmin[p] = abs_bits(dminf);
      pos[p] = mn[p] <= dmin[p] ? argmin : first_mn;
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    auto dk = [&](int g) { return abs_bits(__dsub_rn(S.glk[g], qk[p])); };
    int g;
    uint64_t best;
    if (mn[p] <= dmin[p]) {  // best == dmin: the leftmost group within dmin, member argmin
      if (dkL[p] <= dmin[p]) {
        g = start[p] - 1;
        while (g > 0 && dk(g - 1) <= dmin[p]) --g;
      } else {
        g = start[p];
      }
      best = dmin[p];
    } else {                 // best == mn: the leftmost nearest group, first member within mn
      if (dkL[p] == mn[p]) {
        g = start[p] - 1;
        while (g > 0 && dk(g - 1) == mn[p]) --g;
      } else {
        g = start[p];
      }
      best = mn[p];
    }
    out_best[p] = best;
    out_rec[p] = S.gidx[S.gstart[g] + pos[p]];
  }
}

// blocks / waves of compute.block_count / wave_count with a flag for u64
// overflow: the reference's Python path computes them in unbounded integers
// (compute.py:78-106), so a product past 2^64 is reported, not wrapped.
__device__ __forceinline__ bool predict_point_checked(const TablesDev& t, int c, uint64_t b,
                                                      uint64_t m, uint64_t n, uint64_t k,
                                                      double base, PointResult* r) {
  if (t.rowblock[c]) {
    r->blocks = ceil_div_c(t, c, 0, b * k, t.tile_m[c]);  // b, k < 2^32: no overflow
  } else {
    const uint64_t cm = ceil_div_c(t, c, 0, m, t.tile_m[c]), cn = ceil_div_c(t, c, 1, n, t.tile_n[c]);
    const uint64_t sk = t.split_k[c];
    uint64_t p;
    if (((b | cm | cn | sk) >> 32) == 0) {  // the usual case: two exact 32x32 products
      const uint64_t p1 = b * cm, p2 = cn * sk;
      if (__umul64hi(p1, p2)) return false;
      p = p1 * p2;
    } else {
      const uint64_t f[3] = {cm, cn, sk};
      p = b;
      bool over = false;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        over |= __umul64hi(p, f[i]) != 0;
        p *= f[i];
      }
      if (over) return false;
    }
    r->blocks = p;
  }
  const uint64_t bpw = t.bpw[c];
  if (r->blocks + bpw - 1 < r->blocks) return false;
  r->waves = ceil_div_c(t, c, 2, r->blocks, bpw);
  r->lat = __dmul_rn(base, wave_scale(t, c, r->waves));
  return true;
}

__device__ __forceinline__ uint32_t waves_u32(uint64_t w) {
  return w > 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(w);  // saturated (detail has the value)
}

template <int NEARK>  // 0 general sweep, 1 sweep + tie mask (G <= 32), 2 one class,
                      // 3 one class by rows (u32 masks), 4 by rows (u64 masks)
__global__ void __launch_bounds__(kThreads, PTS_MINB) points_kernel(TablesDev t, const uint4* __restrict__ shapes,
                                                          int64_t n, LogSource L,
                                                          double* __restrict__ out_lat,
                                                          int32_t* __restrict__ out_curve,
                                                          uint32_t* __restrict__ out_waves,
                                                          int8_t* __restrict__ out_match,
                                                          int32_t* __restrict__ out_record,
                                                          double* __restrict__ out_dist,
                                                          double* __restrict__ out_detail) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr bool kRows = NEARK >= 3;
  const int NR = kRows ? t.rw_n : 0, NCl = kRows ? t.cl_n : 0;
  const int NP = kRows ? t.rw_off[NR] : 0;
  double2* lr = reinterpret_cast<double2*>(smem);
  const int NLR = NR * (NCl + 1);
  uint64_t* rmask = reinterpret_cast<uint64_t*>(lr + NLR);
  uint64_t* cmask = rmask + NR;
  double* rlm = reinterpret_cast<double*>(cmask + NCl);
  double* cln = rlm + NR;                        // padded with +inf to pow2_above(NCl)
  const int NClp = kRows ? pow2_above(NCl) : 0;
  double* lm = cln + NClp;
  const int CMs = kRows ? 0 : t.CM;  // the row form needs no member list
  double* ln = lm + CMs;
  double* glk = ln + CMs;                        // padded with +inf to pow2_above(G)
  const int Gp = pow2_above(t.G);
  int32_t* gcls = reinterpret_cast<int32_t*>(glk + Gp);
  int32_t* gstart = gcls + t.G;
  int32_t* cstart = gstart + t.G;
  int32_t* csize = cstart + t.NC;
  int32_t* gidx = csize + t.NC;
  int32_t* roff = gidx + t.R;
  int32_t* rpos = roff + NR + 1;
  for (int j = threadIdx.x; j < NR; j += blockDim.x) {
    rmask[j] = t.rw_mask[j];
    rlm[j] = t.rw_lm[j];
  }
  const double INF = __longlong_as_double(0x7FF0000000000000ll);
  for (int j = threadIdx.x; j < NCl; j += blockDim.x) cmask[j] = t.cl_mask[j];
  for (int j = threadIdx.x; j < NClp; j += blockDim.x) cln[j] = j < NCl ? t.cl_ln[j] : INF;
  for (int j = threadIdx.x; j <= NR && kRows; j += blockDim.x) roff[j] = t.rw_off[j];
  for (int j = threadIdx.x; j < NLR; j += blockDim.x)
    lr[j] = reinterpret_cast<const double2*>(t.rw_lr)[j];
  for (int j = threadIdx.x; j < NP; j += blockDim.x) rpos[j] = t.rw_pos[j];
  for (int j = threadIdx.x; j < CMs; j += blockDim.x) {
    lm[j] = t.cls_lm[j];
    ln[j] = t.cls_ln[j];
  }
  for (int j = threadIdx.x; j < Gp; j += blockDim.x) glk[j] = j < t.G ? t.grp_lk[j] : INF;
  for (int j = threadIdx.x; j < t.G; j += blockDim.x) {
    gcls[j] = t.grp_class[j];
    gstart[j] = t.grp_start[j];
  }
  for (int j = threadIdx.x; j < t.NC; j += blockDim.x) {
    cstart[j] = t.cls_start[j];
    csize[j] = t.cls_size[j];
  }
  for (int j = threadIdx.x; j < t.R; j += blockDim.x) gidx[j] = t.g_idx[j];
  uint32_t* stags = reinterpret_cast<uint32_t*>(rpos + NP);
  const int ntag = t.xh_mask >= 0 && t.xh_mask < kTagSmemSlots ? t.xh_mask + 1 : 0;
  for (int j = threadIdx.x; j < ntag; j += blockDim.x) stags[j] = t.xh_tags[j];
  const uint32_t* tags = ntag ? stags : t.xh_tags;
  __syncthreads();
  const PointSmem S{lm, ln, glk, gcls, gstart, cstart, csize, gidx};
  const RowSmem W{rlm, cln, rmask, cmask, roff, rpos, lr, NR, NCl};
  // warp-uniform trip count (every lane runs every iteration, the tail lanes
  // idle), so the warp can be reconverged before the shared prediction tail.
  // A warp takes 32 * P consecutive ops per iteration, P per lane (op p of
  // lane l = base + 32 p + l: coalesced), whose nearest searches run
  // interleaved (independent FP64 chains per row step)
  constexpr int P = NEARK >= 2 ? kPointsPerLane : 1;
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * P;
  for (int64_t base = (blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31)) * P; base < n;
       base += stride) {
    int64_t idx[P];
    uint4 sh[P];
    int ci[P], rec[P];
    bool zero[P], hit[P], logs[P];
    double qm[P], qn[P], qk[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      idx[p] = base + 32 * p + lane;
      sh[p] = idx[p] < n ? shapes[idx[p]] : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const uint4 s = sh[p];
      const QueryLogs ql = query_logs(L, s);
      ci[p] = -1;
      rec[p] = -1;
      // divergent steps (probe loops, searches) are followed by explicit
      // warp reconvergence: without it the lanes leave a loop at different
      // trips and run the following nearest search in separate passes
      zero[p] = s.x == 0 || s.y == 0 || s.z == 0 || s.w == 0;
#if PTS_VARIANT == 3
      hit[p] = false;  // diagnostic build: no exact lookup
#else
      hit[p] = !zero[p] && (t.xh_mask >= 0 ? exact_hash(t, tags, s, &ci[p], &rec[p])
                                           : exact_lookup(t, s.x, s.y, s.z, s.w, &ci[p], &rec[p]));
#endif
      qm[p] = ql.m;
      qn[p] = ql.n;
      qk[p] = ql.k;
      logs[p] = !zero[p] && !hit[p] && t.R > 0 && ql.ok;
#if PTS_VARIANT == 4
      qm[p] = double(s.y); qn[p] = double(s.z); qk[p] = double(s.w);  // diagnostic build: no log2 loads
#endif
      __syncwarp();
    }
    // the nearest search runs in every lane (exact hits and invalid ops are
    // rare; the warp would run it for the others anyway) so it can keep the
    // warp converged; only the lanes that need it keep its answer
    uint64_t best[P];
    int nrec[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      best[p] = 0;
      nrec[p] = -1;
    }
#if PTS_VARIANT == 1 || PTS_VARIANT == 5
#pragma unroll
    for (int p = 0; p < P; ++p) nrec[p] = int(sh[p].x) & 7;  // diagnostic build: no nearest search
#else
    if (t.R > 0) {
      if constexpr (NEARK >= 2) {
        nearest_point_one_class<NEARK - 2, P>(t, S, W, qm, qn, qk, nrec, best);
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p) nrec[p] = nearest_point<NEARK == 1>(t, S, qm[p], qn[p], qk[p], &best[p]);
      }
    }
#endif
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int64_t i = idx[p];
      const uint4 s = sh[p];
      int c = ci[p], rc = rec[p];
      int8_t match = -1;
      double dist = 0.0;
      if (zero[p]) {
        match = -2;  // invalid coordinate
      } else if (hit[p]) {
        match = 0;
      } else if (t.R > 0) {
        if (!logs[p]) {
          match = -2;  // no host log2 for this coordinate
        } else {
          rc = nrec[p];
          c = t.cand_curve[rc];
          dist = __longlong_as_double(static_cast<long long>(best[p]));
          match = 1;
        }
      }
      __syncwarp();
      PointResult r;
      double thr = 0.0, bse = 0.0;
#if PTS_VARIANT == 2 || PTS_VARIANT == 5
      r.lat = qm[p] + qk[p]; r.waves = s.x;  // diagnostic build: no prediction tail
      if (false) {
#else
      if (c >= 0) {
#endif
        const double nd = __ull2double_rn(uint64_t(s.w));
        thr = interp_thr(t, c, nd);
        bse = base_from_thr(t, c, nd, thr);
        if (!predict_point_checked(t, c, s.x, s.y, s.z, s.w, bse, &r)) {
          match = -3;  // block count past 2^64
          c = -1;
        }
      }
      if (i >= n) continue;
      if (out_record) out_record[i] = rc;
      if (out_dist) out_dist[i] = dist;
      if (out_match) out_match[i] = match;
      if (c < 0) {
        out_lat[i] = qnan();
        if (out_curve) out_curve[i] = -1;
        if (out_waves) out_waves[i] = 0;
        if (out_detail)
          for (int j = 0; j < 4; ++j) out_detail[4 * i + j] = qnan();
        continue;
      }
      out_lat[i] = r.lat;
      if (out_curve) out_curve[i] = c;
      if (out_waves) out_waves[i] = waves_u32(r.waves);
      if (out_detail) {  // Prediction.components: base_us, new_throughput, wave_scale, waves
        out_detail[4 * i] = bse;
        out_detail[4 * i + 1] = thr;
        out_detail[4 * i + 2] = wave_scale(t, c, r.waves);
        out_detail[4 * i + 3] = __ull2double_rn(r.waves);
      }
    }
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
    PointResult r;
    double thr = 0.0, base = 0.0;
    bool ok = c >= 0 && c < t.C && curve_valid(t, c) && s.x && s.y && s.z && s.w;
    if (ok) {
      const double nd = __ull2double_rn(uint64_t(s.w));
      thr = interp_thr(t, c, nd);
      base = base_from_thr(t, c, nd, thr);
      ok = predict_point_checked(t, c, s.x, s.y, s.z, s.w, base, &r);
    }
    if (!ok) {
      out_lat[i] = qnan();
      if (out_waves) out_waves[i] = 0;
      if (out_detail)
        for (int j = 0; j < 4; ++j) out_detail[4 * i + j] = qnan();
      continue;
    }
    out_lat[i] = r.lat;
    if (out_waves) out_waves[i] = waves_u32(r.waves);
    if (out_detail) {  // Prediction.components: base_us, new_throughput, wave_scale, waves
      out_detail[4 * i] = base;
      out_detail[4 * i + 1] = thr;
      out_detail[4 * i + 2] = wave_scale(t, c, r.waves);
      out_detail[4 * i + 3] = __ull2double_rn(r.waves);
    }
  }
}

}  // namespace

int launch_points(const TablesDev& t, const uint32_t* shapes, int64_t n, const LogSource& logs,
                  double* out_lat, int32_t* out_curve, uint32_t* out_waves, int8_t* out_match,
                  int32_t* out_record, double* out_dist, double* out_detail, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool one = t.NC == 1 && t.lowest_wins;
  const bool rows = one && t.rw_n > 0;
  const int64_t NR = rows ? t.rw_n : 0, NCl = rows ? t.cl_n : 0;
  const int64_t smem = 16ll * NR * (NCl + 1) + 16ll * NR + 8ll * NCl + (rows ? 8ll * pow2_above(int(NCl)) : 0) +
                       (rows ? 0 : 16ll * t.CM) + 8ll * pow2_above(t.G) + 8ll * t.G +
                       8ll * t.NC + 4ll * t.R + (rows ? 4ll * (NR + 1 + t.CM) : 0) +
                       (t.xh_mask >= 0 && t.xh_mask < kTagSmemSlots ? 4ll * (t.xh_mask + 1) : 0) + 64;
  auto* fn = rows ? (t.rw_n <= 32 && t.cl_n <= 32 ? points_kernel<3> : points_kernel<4>)
             : one ? points_kernel<2>
             : t.G <= 32 ? points_kernel<1> : points_kernel<0>;
  if (smem > 227 * 1024) return int(cudaErrorInvalidValue);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return int(e);
  }
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(sm_count()) * 8));
  fn<<<nb, kThreads, smem, s>>>(t, reinterpret_cast<const uint4*>(shapes), n, logs, out_lat,
                                out_curve, out_waves, out_match, out_record, out_dist, out_detail);
  return int(cudaGetLastError());
}

int launch_points_curve(const TablesDev& t, const uint32_t* shapes, const int32_t* curves, int64_t n,
                        double* out_lat, uint32_t* out_waves, double* out_detail, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(sm_count()) * 16));
  points_curve_kernel<<<nb, kThreads, 0, s>>>(t, reinterpret_cast<const uint4*>(shapes), curves, n,
                                             out_lat, out_waves, out_detail);
  return int(cudaGetLastError());
}

}  // namespace pm2l
