// Host-side planner: turns the reference's flat tables (PreparedGrid.tables(),
// pm2lat/nascache.py:174-241) into the HBM layout the sm_100a kernels use,
// and builds the per-call grid description (axis values, host libm log2 of
// every axis value, exact-hit fix-up list).
//
// Nothing here computes a latency; it only reorganises inputs.  log2 comes
// from the host libm, exactly as the Cython kernel (_kernels.pyx:101,104,112)
// and the Python resolver's math.log2 (compute.py:261) obtain it — device
// log2 differs by an ulp on some integers and is never used.
#include <algorithm>
#include <limits>
#include <array>
#include <cmath>
#include <cstring>
#include <utility>
#include <vector>
#include <map>
#include <numeric>
#include <string>
#include <unordered_map>

#include "../../include/pm2l.h"
#include "pm2l_internal.h"

namespace pm2l {
namespace {

// Append-only byte blob with 256-byte aligned sections; section pointers are
// recorded as offsets and rebased onto the device copy later.
class Blob {
 public:
  template <class T>
  const T* add(const T* src, size_t count) {
    size_t off = (bytes_.size() + 255) & ~size_t(255);
    bytes_.resize(off + count * sizeof(T));
    if (count) std::memcpy(bytes_.data() + off, src, count * sizeof(T));
    return reinterpret_cast<const T*>(off);
  }
  template <class T>
  const T* add(const std::vector<T>& v) { return add(v.data(), v.size()); }
  // trailing slack: 16-byte bulk copies of the last section may read past it
  std::vector<uint8_t>& bytes() {
    bytes_.resize(((bytes_.size() + 255) & ~size_t(255)) + 256);
    return bytes_;
  }

 private:
  std::vector<uint8_t> bytes_;
};

template <class T>
const T* shift(const T* off, const void* base) {
  return reinterpret_cast<const T*>(static_cast<const uint8_t*>(base) +
                                    reinterpret_cast<uintptr_t>(off));
}

}  // namespace

std::string build_tables(const pm2l_tables_view* v, TablesHost* out) {
  if (!v) return "null tables view";
  const int64_t R = v->n_records, C = v->n_curves;
  if (R < 0 || C < 0) return "negative table size";
  if (R > (int64_t(1) << 30) || C > (int64_t(1) << 30)) return "tables too large";
  if (R > 0 && (!v->log_m || !v->log_n || !v->log_k || !v->cand_curve || !v->exact_curve))
    return "missing candidate arrays";
  if (R > 0 && !v->exact_keys && !v->exact_coords) return "need exact_keys or exact_coords";
  if (!v->sample_offsets) return "missing sample_offsets";
  if (C > 0 && (!v->ref_dim || !v->ref_dur || !v->ref_thr || !v->ref_waves || !v->tile_m ||
                !v->tile_n || !v->split_k || !v->blocks_per_wave || !v->family_rowblock))
    return "missing curve arrays";
  if (v->sample_offsets[0] != 0) return "sample_offsets[0] must be 0";
  for (int64_t c = 0; c < C; ++c)
    if (v->sample_offsets[c + 1] < v->sample_offsets[c]) return "sample_offsets not monotone";
  const int64_t S = v->sample_offsets[C];
  if (S > 0 && (!v->sample_dims || !v->sample_thrs)) return "missing samples";
  if (S >= (int64_t(1) << 31)) return "too many samples";

  std::vector<uint8_t> referenced(C, 0);
  auto check_curve = [&](int64_t c) -> bool {
    if (c < -1 || c >= C) return false;
    if (c >= 0) referenced[c] = 1;
    return true;
  };
  for (int64_t i = 0; i < R; ++i)
    if (!check_curve(v->cand_curve[i]) || !check_curve(v->exact_curve[i]))
      return "curve index out of range";
  int32_t all_gemm = 1, n_ref = 0, n_rowblock = 0;
  for (int64_t c = 0; c < C; ++c) {
    if (!referenced[c]) continue;
    if (v->sample_offsets[c + 1] - v->sample_offsets[c] < 1)
      return "a referenced curve has no samples";
    if (v->tile_m[c] < 1 || v->blocks_per_wave[c] < 1) return "tile_m and blocks_per_wave must be >= 1";
    if (!v->family_rowblock[c] && (v->tile_n[c] < 1 || v->split_k[c] < 1))
      return "tile_n and split_k must be >= 1";
    if (!(v->ref_dim[c] > 0) || !(v->ref_waves[c] > 0)) return "ref_dim/ref_waves must be > 0";
    if (v->family_rowblock[c]) all_gemm = 0;
    ++n_ref;
    n_rowblock += v->family_rowblock[c] ? 1 : 0;
  }
  for (int64_t i = 0; i < R; ++i)
    if (!std::isfinite(v->log_m[i]) || !std::isfinite(v->log_n[i]) || !std::isfinite(v->log_k[i]))
      return "candidate logs must be finite";

  // --- k-groups: distinct log_k values ascending, members in scan order
  std::vector<int32_t> order(R);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return v->log_k[a] < v->log_k[b]; });
  std::vector<double> grp_lk, g_lm(R), g_ln(R);
  std::vector<int32_t> grp_start, grp_size, g_idx(R);
  int64_t max_group = 0;
  for (int64_t p = 0; p < R; ++p) {
    int32_t i = order[p];
    if (p == 0 || v->log_k[i] != grp_lk.back()) {
      grp_lk.push_back(v->log_k[i]);
      grp_start.push_back(int32_t(p));
      grp_size.push_back(0);
    }
    grp_size.back() += 1;
    max_group = std::max<int64_t>(max_group, grp_size.back());
    g_lm[p] = v->log_m[i];
    g_ln[p] = v->log_n[i];
    g_idx[p] = i;  // stable sort keeps ascending scan order inside a group
  }
  // --- member classes (groups with identical (lm, ln) member sequences)
  std::vector<int32_t> grp_class(grp_lk.size()), cls_start, cls_size;
  std::vector<double> cls_lm, cls_ln;
  {
    std::map<std::vector<std::pair<uint64_t, uint64_t>>, int32_t> seen;
    for (size_t gi = 0; gi < grp_lk.size(); ++gi) {
      std::vector<std::pair<uint64_t, uint64_t>> sig;
      for (int32_t p = grp_start[gi]; p < grp_start[gi] + grp_size[gi]; ++p) {
        uint64_t a, b;
        std::memcpy(&a, &g_lm[p], 8);
        std::memcpy(&b, &g_ln[p], 8);
        sig.emplace_back(a, b);
      }
      auto it = seen.find(sig);
      if (it == seen.end()) {
        const int32_t id = int32_t(cls_start.size());
        cls_start.push_back(int32_t(cls_lm.size()));
        cls_size.push_back(grp_size[gi]);
        for (int32_t p = grp_start[gi]; p < grp_start[gi] + grp_size[gi]; ++p) {
          cls_lm.push_back(g_lm[p]);
          cls_ln.push_back(g_ln[p]);
        }
        it = seen.emplace(std::move(sig), id).first;
      }
      grp_class[gi] = it->second;
    }
  }
  std::vector<int32_t> cand_curve(R), g_curve(R);
  for (int64_t i = 0; i < R; ++i) cand_curve[i] = int32_t(v->cand_curve[i]);
  for (int64_t p = 0; p < R; ++p) g_curve[p] = cand_curve[g_idx[p]];

  // --- exact records, unpacked and sorted by (b, m, n, k)
  std::vector<std::array<uint64_t, 6>> ex(R);
  for (int64_t i = 0; i < R; ++i) {
    uint64_t b, m, n, k;
    if (v->exact_coords) {
      b = v->exact_coords[4 * i]; m = v->exact_coords[4 * i + 1];
      n = v->exact_coords[4 * i + 2]; k = v->exact_coords[4 * i + 3];
    } else {
      const uint64_t key = v->exact_keys[i];  // nascache.py:188 packing
      b = key >> 48; m = (key >> 32) & 0xFFFF; n = (key >> 16) & 0xFFFF; k = key & 0xFFFF;
    }
    ex[i] = {b, m, n, k, uint64_t(int64_t(v->exact_curve[i])), uint64_t(i)};
  }
  std::stable_sort(ex.begin(), ex.end(), [](const auto& a, const auto& b) {
    return std::lexicographical_compare(a.begin(), a.begin() + 4, b.begin(), b.begin() + 4);
  });
  std::vector<uint64_t> ex_coord(4 * R);
  std::vector<int32_t> ex_curve(R), ex_rec(R);
  for (int64_t i = 0; i < R; ++i) {
    for (int j = 0; j < 4; ++j) ex_coord[4 * i + j] = ex[i][j];
    ex_curve[i] = int32_t(int64_t(ex[i][4]));
    ex_rec[i] = int32_t(ex[i][5]);
  }
  // two exact records of one shape naming different kernels are the
  // reference resolver's AmbiguousConfig (compute.py:227-234); the same
  // kernel twice is kept once in the device planner's copy below
  for (int64_t i = 1; i < R; ++i)
    if (std::equal(ex[i].begin(), ex[i].begin() + 4, ex[i - 1].begin()) && ex[i][4] != ex[i - 1][4])
      return "ambiguous exact records: one shape, two kernels";
  // the device planner's copy: unique shapes sorted by (m, n, b, k), so the
  // records of one (m, n) row are one contiguous range
  std::vector<std::array<uint64_t, 6>> exm;
  for (int64_t i = 0; i < R; ++i)
    if (i == 0 || !std::equal(ex[i].begin(), ex[i].begin() + 4, ex[i - 1].begin())) exm.push_back(ex[i]);
  std::stable_sort(exm.begin(), exm.end(), [](const auto& a, const auto& b) {
    const std::array<uint64_t, 4> ka = {a[1], a[2], a[0], a[3]}, kb = {b[1], b[2], b[0], b[3]};
    return ka < kb;
  });
  std::vector<uint64_t> exm_coord(4 * exm.size());
  std::vector<int32_t> exm_curve(exm.size());
  for (size_t i = 0; i < exm.size(); ++i) {
    for (int j = 0; j < 4; ++j) exm_coord[4 * i + j] = exm[i][j];
    exm_curve[i] = int32_t(int64_t(exm[i][4]));
  }

  // u32 division magic (Granlund & Montgomery, PLDI'94, fig. 4.1): for every
  // 32-bit n, n / d == (t + ((n - t) >> sh1)) >> sh2 with t = umulhi(m, n)
  std::vector<uint32_t> dv_m(3 * C, 0), dv_s(3 * C, 0);
  for (int64_t c = 0; c < C; ++c) {
    const uint64_t divs[3] = {v->tile_m[c], v->tile_n[c], v->blocks_per_wave[c]};
    for (int j = 0; j < 3; ++j) {
      const uint64_t d = divs[j];
      if (d < 1 || d > 0xFFFFFFFFull) continue;  // not valid: generic u64 division
      int l = 0;
      while ((uint64_t(1) << l) < d) ++l;
      const uint64_t m = ((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1;
      const uint32_t sh1 = l < 1 ? l : 1, sh2 = l > 1 ? l - 1 : 0;
      dv_m[3 * c + j] = uint32_t(m);
      dv_s[3 * c + j] = sh1 | (sh2 << 8) | (1u << 16);
    }
  }
  // wave classes
  std::vector<int32_t> wc_of(C, -1), wc_rep;
  {
    std::map<std::array<uint64_t, 6>, int32_t> seen;
    for (int64_t c = 0; c < C; ++c) {
      if (v->sample_offsets[c + 1] <= v->sample_offsets[c]) continue;
      uint64_t rw;
      std::memcpy(&rw, &v->ref_waves[c], 8);
      const std::array<uint64_t, 6> key = {uint64_t(v->family_rowblock[c] ? 1 : 0), v->tile_m[c],
                                           v->tile_n[c], v->split_k[c], v->blocks_per_wave[c], rw};
      auto it = seen.find(key);
      if (it == seen.end()) {
        it = seen.emplace(key, int32_t(wc_rep.size())).first;
        wc_rep.push_back(int32_t(c));
      }
      wc_of[c] = it->second;
    }
  }
  std::vector<int32_t> g_cw(2 * R);
  for (int64_t p = 0; p < R; ++p) {
    g_cw[2 * p] = g_curve[p];
    g_cw[2 * p + 1] = g_curve[p] >= 0 ? wc_of[g_curve[p]] : -1;
  }
  std::vector<WcParam> wcp(wc_rep.size());
  for (size_t w = 0; w < wc_rep.size(); ++w) {
    const int32_t c = wc_rep[w];
    WcParam& q = wcp[w];
    q.tm = v->tile_m[c]; q.tn = v->tile_n[c]; q.sk = v->split_k[c]; q.bpw = v->blocks_per_wave[c];
    q.rw = v->ref_waves[c];
    for (int j = 0; j < 3; ++j) { q.dm[j] = dv_m[3 * c + j]; q.ds[j] = dv_s[3 * c + j]; }
    if (v->family_rowblock[c]) {
      // row-block classes never divide by tile_n: slot 1 carries
      // tile_m * blocks_per_wave instead, so the lookup kernel computes
      // waves = ceil(ceil(b*k / tm) / bpw) = ceil(b*k / (tm * bpw)) with one
      // magic division (grid.cu rb_scale); ds[1] = 0 when it does not fit
      q.tn = 0; q.dm[1] = 0; q.ds[1] = 0;
      const uint64_t d = q.tm * q.bpw;
      if (q.tm <= 0xFFFFFFFFull && q.bpw <= 0xFFFFFFFFull && d <= 0xFFFFFFFFull) {
        int l = 0;
        while ((uint64_t(1) << l) < d) ++l;
        q.tn = d;
        q.dm[1] = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
        q.ds[1] = uint32_t(l < 1 ? l : 1) | (uint32_t(l > 1 ? l - 1 : 0) << 8) | (1u << 16);
      }
    }
  }
  // the same parameters per curve (zero for a curve without samples): one
  // load instead of the wc_of -> wcp chain where a kernel stages them by curve
  std::vector<WcParam> wcp_c(static_cast<size_t>(C));
  for (int64_t c = 0; c < C; ++c)
    if (wc_of[c] >= 0) wcp_c[c] = wcp[size_t(wc_of[c])];
  std::vector<int32_t> s_off(C + 1);
  for (int64_t c = 0; c <= C; ++c) s_off[c] = int32_t(v->sample_offsets[c]);
  std::vector<uint8_t> rowblock(C);
  for (int64_t c = 0; c < C; ++c) rowblock[c] = v->family_rowblock[c] ? 1 : 0;

  // --- explicit-descriptor exact hash (records whose coordinates fit u32;
  // the first record of each shape in the caller's order, as a linear scan
  // of the exact arrays finds it)
  int32_t xh_mask = -1;
  std::vector<uint4> xh_key;
  std::vector<int2> xh_val;
  std::vector<uint32_t> xh_tags;
  if (R > 0) {
    int64_t cap = 16;
    while (cap < 2 * R) cap <<= 1;
    xh_mask = int32_t(cap - 1);
    xh_key.assign(size_t(cap), uint4{0, 0, 0, 0});
    xh_val.assign(size_t(cap), int2{-1, -1});
    xh_tags.assign(size_t(cap), 0u);
    // ex is sorted by shape, stable: equal shapes keep caller order
    for (int64_t i = 0; i < R; ++i) {
      const auto& e = ex[i];
      if (i > 0 && std::equal(e.begin(), e.begin() + 4, ex[i - 1].begin())) continue;
      if ((e[0] | e[1] | e[2] | e[3]) > 0xFFFFFFFFull || !e[0] || !e[1] || !e[2] || !e[3])
        continue;  // cannot equal a u32 descriptor with coordinates >= 1
      const uint4 key{uint32_t(e[0]), uint32_t(e[1]), uint32_t(e[2]), uint32_t(e[3])};
      uint32_t h = xh_hash(key.x, key.y, key.z, key.w) & uint32_t(xh_mask);
      while (xh_key[h].x) h = (h + 1) & uint32_t(xh_mask);
      xh_key[h] = key;
      xh_val[h] = int2{int32_t(int64_t(e[4])), int32_t(e[5])};
      xh_tags[h] = xh_tag(key.x, key.y, key.z, key.w);
    }
  }
  // --- row decomposition of class 0 (one member class)
  std::vector<double> rw_lm, cl_ln;
  std::vector<uint64_t> rw_mask, cl_mask;
  std::vector<int32_t> rw_off, rw_pos;
  std::vector<double> rw_lr;
  if (cls_start.size() == 1) {
    const int32_t CMm = cls_size[0];
    auto bits = [](double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; };
    std::vector<double> lms(cls_lm.begin(), cls_lm.begin() + CMm);
    std::vector<double> lns(cls_ln.begin(), cls_ln.begin() + CMm);
    std::vector<double> rows = lms, cols = lns;
    std::sort(rows.begin(), rows.end());
    rows.erase(std::unique(rows.begin(), rows.end(),
                           [&](double a, double b) { return bits(a) == bits(b); }), rows.end());
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end(),
                           [&](double a, double b) { return bits(a) == bits(b); }), cols.end());
    bool ok = rows.size() <= 64 && cols.size() <= 64 && !rows.empty();
    std::vector<std::pair<int32_t, int32_t>> seen;  // deduplicated (row, col) in scan order
    std::vector<int32_t> first_pos;
    for (int32_t j = 0; ok && j < CMm; ++j) {
      const int32_t r = int32_t(std::lower_bound(rows.begin(), rows.end(), lms[j]) - rows.begin());
      const int32_t c = int32_t(std::lower_bound(cols.begin(), cols.end(), lns[j]) - cols.begin());
      const std::pair<int32_t, int32_t> rc{r, c};
      if (std::find(seen.begin(), seen.end(), rc) != seen.end()) continue;  // duplicate
      if (!seen.empty() && !(seen.back() < rc)) ok = false;  // not (row, col)-lexicographic
      seen.push_back(rc);
      first_pos.push_back(j);
    }
    if (ok) {
      rw_lm = rows;
      cl_ln = cols;
      rw_mask.assign(rows.size(), 0);
      cl_mask.assign(cols.size(), 0);
      rw_off.assign(rows.size() + 1, 0);
      for (const auto& rc : seen) {
        rw_mask[rc.first] |= uint64_t(1) << rc.second;
        cl_mask[rc.second] |= uint64_t(1) << rc.first;
        rw_off[rc.first + 1] += 1;
      }
      for (size_t i = 0; i < rows.size(); ++i) rw_off[i + 1] += rw_off[i];
      rw_pos = first_pos;  // seen is lexicographic: row-major, columns ascending
      // nearest present column of each row on either side of each column
      // insertion point pc: (log n of the highest present column < pc, of
      // the lowest present column >= pc), -inf / +inf where the side is
      // empty (so qn - lower and upper - qn are +inf there)
      const size_t NCp = cols.size() + 1;
      const double inf = std::numeric_limits<double>::infinity();
      rw_lr.assign(2 * rows.size() * NCp, inf);
      for (size_t e = 0; e < rw_lr.size(); e += 2) rw_lr[e] = -inf;
      for (size_t i = 0; i < rows.size(); ++i)
        for (size_t pc = 0; pc < NCp; ++pc) {
          for (size_t j = pc; j-- > 0;)
            if (rw_mask[i] >> j & 1) { rw_lr[2 * (i * NCp + pc)] = cols[j]; break; }
          for (size_t j = pc; j < cols.size(); ++j)
            if (rw_mask[i] >> j & 1) { rw_lr[2 * (i * NCp + pc) + 1] = cols[j]; break; }
        }
    }
  }

  Blob blob;
  TablesDev& t = out->dev_offsets;
  t = TablesDev{};
  t.R = int32_t(R); t.C = int32_t(C); t.G = int32_t(grp_lk.size());
  t.n_exact = int32_t(R); t.all_gemm = all_gemm; t.n_samples = int32_t(S);
  t.all_rowblock = n_ref > 0 && n_rowblock == n_ref ? 1 : 0;
  {
    // log2 is injective on integers below 2^44 at double precision, so equal
    // candidate logs there imply equal coordinates (grid.cu one-class path)
    bool small = true;
    for (int64_t i = 0; i < R; ++i)
      small = small && v->log_m[i] < 44.0 && v->log_n[i] < 44.0 && v->log_k[i] < 44.0;
    t.lowest_wins = small ? 1 : 0;
  }
  {
    // every member of the one class at one (log m, log n): batch values are
    // the only difference, so the first member (scan order) attains every
    // row's minimum (grid_single.cu)
    bool one = cls_start.size() == 1 && !cls_lm.empty();
    for (size_t j = 1; one && j < cls_lm.size(); ++j)
      one = std::memcmp(&cls_lm[j], &cls_lm[0], 8) == 0 && std::memcmp(&cls_ln[j], &cls_ln[0], 8) == 0;
    t.single_mn = one ? 1 : 0;
  }
  t.ref_dim = blob.add(v->ref_dim, C);
  t.ref_dur = blob.add(v->ref_dur, C);
  t.ref_thr = blob.add(v->ref_thr, C);
  t.ref_waves = blob.add(v->ref_waves, C);
  t.tile_m = blob.add(v->tile_m, C);
  t.tile_n = blob.add(v->tile_n, C);
  t.split_k = blob.add(v->split_k, C);
  t.bpw = blob.add(v->blocks_per_wave, C);
  t.dv_m = blob.add(dv_m);
  t.dv_s = blob.add(dv_s);
  t.NW = int32_t(wc_rep.size());
  t.wc_of = blob.add(wc_of);
  t.wc_rep = blob.add(wc_rep);
  t.rowblock = blob.add(rowblock);
  t.s_off = blob.add(s_off);
  t.s_dims = blob.add(v->sample_dims, S);
  t.s_thrs = blob.add(v->sample_thrs, S);
  t.g_lm = blob.add(g_lm);
  t.g_ln = blob.add(g_ln);
  t.g_idx = blob.add(g_idx);
  t.cand_curve = blob.add(cand_curve);
  t.g_curve = blob.add(g_curve);
  t.g_cw = blob.add(g_cw);
  t.wcp = blob.add(wcp);
  t.wcp_c = blob.add(wcp_c);
  t.grp_lk = blob.add(grp_lk);
  t.grp_start = blob.add(grp_start);
  {
    std::vector<int32_t> gc0(grp_start.size());
    for (size_t gi = 0; gi < grp_start.size(); ++gi) gc0[gi] = g_curve[grp_start[gi]];
    t.grp_curve0 = blob.add(gc0);
    std::vector<uint64_t> rk;
    for (int64_t i = 0; i < R; ++i) rk.push_back(ex[i][3]);
    std::sort(rk.begin(), rk.end());
    rk.erase(std::unique(rk.begin(), rk.end()), rk.end());
    t.n_rec_k = int32_t(rk.size());
    t.rec_k = blob.add(rk);
  }
  t.grp_size = blob.add(grp_size);
  t.grp_class = blob.add(grp_class);
  t.NC = int32_t(cls_start.size());
  t.CM = int32_t(cls_lm.size());
  t.cls_start = blob.add(cls_start);
  t.cls_size = blob.add(cls_size);
  t.cls_lm = blob.add(cls_lm);
  t.cls_ln = blob.add(cls_ln);
  t.ex_coord = blob.add(ex_coord);
  t.ex_curve = blob.add(ex_curve);
  t.ex_rec = blob.add(ex_rec);
  t.n_mn = int32_t(exm.size());
  t.ex_mn_coord = blob.add(exm_coord);
  t.ex_mn_curve = blob.add(exm_curve);
  t.xh_mask = xh_mask;
  t.xh_key = blob.add(xh_key);
  t.xh_val = blob.add(xh_val);
  t.xh_tags = blob.add(xh_tags);
  t.rw_n = int32_t(rw_lm.size());
  t.cl_n = int32_t(cl_ln.size());
  t.rw_lm = blob.add(rw_lm);
  t.cl_ln = blob.add(cl_ln);
  t.rw_mask = blob.add(rw_mask);
  t.cl_mask = blob.add(cl_mask);
  t.rw_off = blob.add(rw_off);
  t.rw_pos = blob.add(rw_pos);
  t.rw_lr = blob.add(rw_lr);
  out->blob.swap(blob.bytes());
  out->max_group = max_group;
  return "";
}

TablesDev rebase(const TablesDev& o, const void* base) {
  TablesDev t = o;
  t.ref_dim = shift(o.ref_dim, base); t.ref_dur = shift(o.ref_dur, base);
  t.ref_thr = shift(o.ref_thr, base); t.ref_waves = shift(o.ref_waves, base);
  t.tile_m = shift(o.tile_m, base); t.tile_n = shift(o.tile_n, base);
  t.split_k = shift(o.split_k, base); t.bpw = shift(o.bpw, base);
  t.dv_m = shift(o.dv_m, base); t.dv_s = shift(o.dv_s, base);
  t.wc_of = shift(o.wc_of, base); t.wc_rep = shift(o.wc_rep, base);
  t.rowblock = shift(o.rowblock, base); t.s_off = shift(o.s_off, base);
  t.s_dims = shift(o.s_dims, base); t.s_thrs = shift(o.s_thrs, base);
  t.g_lm = shift(o.g_lm, base); t.g_ln = shift(o.g_ln, base);
  t.g_idx = shift(o.g_idx, base); t.cand_curve = shift(o.cand_curve, base);
  t.g_curve = shift(o.g_curve, base);
  t.g_cw = shift(o.g_cw, base); t.wcp = shift(o.wcp, base);
  t.wcp_c = shift(o.wcp_c, base);
  t.grp_lk = shift(o.grp_lk, base); t.grp_start = shift(o.grp_start, base);
  t.grp_size = shift(o.grp_size, base); t.grp_class = shift(o.grp_class, base);
  t.grp_curve0 = shift(o.grp_curve0, base); t.rec_k = shift(o.rec_k, base);
  t.cls_start = shift(o.cls_start, base); t.cls_size = shift(o.cls_size, base);
  t.cls_lm = shift(o.cls_lm, base); t.cls_ln = shift(o.cls_ln, base);
  t.ex_coord = shift(o.ex_coord, base); t.ex_curve = shift(o.ex_curve, base);
  t.ex_rec = shift(o.ex_rec, base);
  t.ex_mn_coord = shift(o.ex_mn_coord, base);
  t.ex_mn_curve = shift(o.ex_mn_curve, base);
  t.xh_key = shift(o.xh_key, base); t.xh_val = shift(o.xh_val, base);
  t.xh_tags = shift(o.xh_tags, base);
  t.rw_lm = shift(o.rw_lm, base); t.cl_ln = shift(o.cl_ln, base);
  t.rw_mask = shift(o.rw_mask, base); t.cl_mask = shift(o.cl_mask, base);
  t.rw_off = shift(o.rw_off, base); t.rw_pos = shift(o.rw_pos, base);
  t.rw_lr = shift(o.rw_lr, base);
  return t;
}

std::string build_grid(const TablesHost& th, const uint64_t* const axes[4],
                       const int64_t lens[4], int64_t b_lo, int64_t b_hi, GridHost* out) {
  for (int a = 0; a < 4; ++a) {
    if (lens[a] < 0) return "negative axis length";
    if (lens[a] > 0 && !axes[a]) return "null axis array";
    for (int64_t i = 0; i < lens[a]; ++i)
      if (axes[a][i] == 0) return "grid coordinates must be >= 1";
  }
  if (b_lo < 0 || b_hi < b_lo || b_hi > lens[0]) return "batch slice out of range";
  const int64_t nM = lens[1], nN = lens[2], nK = lens[3];
  std::vector<double> logs[3];
  for (int a = 1; a < 4; ++a) {
    logs[a - 1].resize(lens[a]);
    for (int64_t i = 0; i < lens[a]; ++i) logs[a - 1][i] = std::log2(double(axes[a][i]));
  }

  // per k: insertion point of log2(k) among the (ascending) group lk values
  const TablesDev& tt = th.dev_offsets;
  const double* glk = reinterpret_cast<const double*>(
      th.blob.data() + reinterpret_cast<uintptr_t>(tt.grp_lk));
  std::vector<KInfo> kinfo(nK);
  for (int64_t i = 0; i < nK; ++i)
    kinfo[i] = {logs[2][i], int32_t(std::lower_bound(glk, glk + tt.G, logs[2][i]) - glk), 0};

  // k-only part of the one-class nearest argmin (grid.cu, lookup path): per
  // k, the distance mn(k) from log2 k to the nearest k-group, the leftmost
  // group attaining it (gB), and rank(k) in the stable descending order of
  // mn.  A row's cut points are thresholds on that order.  Same IEEE
  // subtraction and |.| as the device (host double, no contraction).
  std::vector<uint32_t> kfast;
  std::vector<uint64_t> mn_sorted;
  std::vector<int32_t> kright;
  const bool fast_ok = tt.G >= 1 && tt.G <= 255 && nK >= 1 && nK <= 65535;
  if (fast_ok) {
    const int G = tt.G;
    std::vector<uint64_t> mn(nK);
    std::vector<int32_t> gB(nK);
    auto dk = [&](int g, double qk) {
      const double d = glk[g] - qk;
      uint64_t u;
      std::memcpy(&u, &d, 8);
      return u & 0x7FFFFFFFFFFFFFFFull;
    };
    for (int64_t i = 0; i < nK; ++i) {
      const double qk = kinfo[i].qk;
      const int start = kinfo[i].start;
      const uint64_t dkL = start > 0 ? dk(start - 1, qk) : ~0ull;
      const uint64_t dkR = start < G ? dk(start, qk) : ~0ull;
      mn[i] = std::min(dkL, dkR);
      int g = start;
      if (start > 0 && dkL == mn[i]) {
        g = start - 1;
        while (g > 0 && dk(g - 1, qk) == mn[i]) --g;
      }
      gB[i] = g;
    }
    kfast.resize(nK);
    mn_sorted.resize(nK);
    for (int64_t k0 = 0; k0 < nK; k0 += kKChunk) {
      const int64_t k1 = std::min<int64_t>(nK, k0 + kKChunk);
      std::vector<int32_t> ord(k1 - k0);
      std::iota(ord.begin(), ord.end(), int32_t(k0));
      std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return mn[a] > mn[b]; });
      for (int64_t r = 0; r < k1 - k0; ++r) {
        const int32_t i = ord[r];
        mn_sorted[k0 + r] = mn[i];
        kfast[i] = uint32_t(r) | (uint32_t(gB[i]) << 16) | (uint32_t(kinfo[i].start) << 24);
      }
    }
    // per (chunk, group): first chunk-local k index whose log2 k lies right
    // of the group (start(ik) > g)
    for (int64_t k0 = 0; k0 < nK; k0 += kKChunk) {
      const int64_t k1 = std::min<int64_t>(nK, k0 + kKChunk);
      for (int g = 0; g < G; ++g) {
        int64_t i = k0;
        while (i < k1 && kinfo[i].start <= g) ++i;
        kright.push_back(int32_t(i - k0));
      }
    }
  }

  // exact-hit fix-ups: every grid point whose (b, m, n, k) equals a recorded
  // shape takes the recorded kernel (_kernels.pyx:107-110) instead of the
  // nearest one.  Axes may contain duplicates (the raw FFI allows it), so
  // each value maps to all of its indices.
  std::unordered_multimap<uint64_t, int64_t> where[4];
  for (int a = 0; a < 4; ++a) {
    int64_t lo = a == 0 ? b_lo : 0, hi = a == 0 ? b_hi : lens[a];
    for (int64_t i = lo; i < hi; ++i) where[a].emplace(axes[a][i], i);
  }
  const TablesDev& t = th.dev_offsets;
  const uint64_t* exc = reinterpret_cast<const uint64_t*>(
      th.blob.data() + reinterpret_cast<uintptr_t>(t.ex_coord));
  const int32_t* exv = reinterpret_cast<const int32_t*>(
      th.blob.data() + reinterpret_cast<uintptr_t>(t.ex_curve));
  std::map<int64_t, std::pair<std::array<uint64_t, 4>, int32_t>> fix;
  for (int32_t r = 0; r < t.n_exact; ++r) {
    const uint64_t* c = exc + 4 * r;
    auto rb = where[0].equal_range(c[0]);
    if (rb.first == rb.second) continue;
    auto rm = where[1].equal_range(c[1]);
    if (rm.first == rm.second) continue;
    auto rn = where[2].equal_range(c[2]);
    if (rn.first == rn.second) continue;
    auto rk = where[3].equal_range(c[3]);
    for (auto ib = rb.first; ib != rb.second; ++ib)
      for (auto im = rm.first; im != rm.second; ++im)
        for (auto jn = rn.first; jn != rn.second; ++jn)
          for (auto ik = rk.first; ik != rk.second; ++ik) {
            int64_t pos = (((ib->second - b_lo) * nM + im->second) * nN + jn->second) * nK +
                          ik->second;
            fix[pos] = {{c[0], c[1], c[2], c[3]}, exv[r]};
          }
  }
  std::vector<int64_t> fix_pos;
  std::vector<uint64_t> fix_coord;
  std::vector<int32_t> fix_curve;
  const int64_t rows = nM * nN, inner = nM * nN * nK;
  std::vector<int32_t> fixr_off(rows + 1, 0);
  std::vector<FixEntry> fixr;
  for (auto& [pos, val] : fix) {
    fix_pos.push_back(pos);
    for (int j = 0; j < 4; ++j) fix_coord.push_back(val.first[j]);
    fix_curve.push_back(val.second);
    const int64_t ib = pos / inner, rem = pos - ib * inner;
    fixr_off[rem / nK + 1] += 1;
  }
  int32_t max_fix_row = 0;
  for (int64_t r = 0; r < rows; ++r) {
    max_fix_row = std::max(max_fix_row, fixr_off[r + 1]);
    fixr_off[r + 1] += fixr_off[r];
  }
  fixr.resize(fix_pos.size());
  {
    std::vector<int32_t> fill(fixr_off.begin(), fixr_off.end() - 1);
    const int32_t* wc_of = reinterpret_cast<const int32_t*>(
        th.blob.data() + reinterpret_cast<uintptr_t>(tt.wc_of));
    for (auto& [pos, val] : fix) {
      const int64_t ib = pos / inner, rem = pos - ib * inner;
      const int64_t row = rem / nK, ik = rem - row * nK;
      const int32_t ci = val.second;
      fixr[fill[row]++] = FixEntry{int32_t(ik), int32_t(ib), ci, ci >= 0 ? wc_of[ci] : -1};
    }
  }

  Blob blob;
  GridDev& g = out->dev_offsets;
  g = GridDev{};
  g.nB = lens[0]; g.nM = nM; g.nN = nN; g.nK = nK; g.b_lo = b_lo; g.b_hi = b_hi;
  g.B = blob.add(axes[0], lens[0]);
  g.M = blob.add(axes[1], nM);
  g.N = blob.add(axes[2], nN);
  g.K = blob.add(axes[3], nK);
  g.logM = blob.add(logs[0]);
  g.logN = blob.add(logs[1]);
  g.logK = blob.add(logs[2]);
  g.kinfo = blob.add(kinfo);
  g.kfast = fast_ok ? blob.add(kfast) : nullptr;
  g.mn_sorted = fast_ok ? blob.add(mn_sorted) : nullptr;
  g.kright = fast_ok ? blob.add(kright) : nullptr;
  g.n_fix = int64_t(fix_pos.size());
  g.fix_pos = blob.add(fix_pos);
  g.fix_coord = blob.add(fix_coord);
  g.fix_curve = blob.add(fix_curve);
  g.fixr_off = blob.add(fixr_off);
  g.fixr = blob.add(fixr);
  g.max_fix_row = max_fix_row;
  g.k_sorted = 1;
  for (int64_t i = 1; i < nK; ++i)
    if (!(axes[3][i - 1] < axes[3][i])) g.k_sorted = 0;
  out->blob.swap(blob.bytes());
  return "";
}

GridDev rebase(const GridDev& o, const void* base) {
  GridDev g = o;
  g.B = shift(o.B, base); g.M = shift(o.M, base); g.N = shift(o.N, base);
  g.K = shift(o.K, base); g.logM = shift(o.logM, base); g.logN = shift(o.logN, base);
  g.logK = shift(o.logK, base); g.kinfo = shift(o.kinfo, base);
  if (o.kfast) {
    g.kfast = shift(o.kfast, base);
    g.mn_sorted = shift(o.mn_sorted, base);
    g.kright = shift(o.kright, base);
  }
  g.fix_pos = shift(o.fix_pos, base);
  g.fix_coord = shift(o.fix_coord, base); g.fix_curve = shift(o.fix_curve, base);
  g.fixr_off = shift(o.fixr_off, base); g.fixr = shift(o.fixr, base);
  return g;
}

}  // namespace pm2l
