// Device helpers shared by the sm_100a kernels: the reference's canonical
// per-point arithmetic (pm2lat/compute.py:78-138, _kernels.pyx:50-73,119-132).
//
// Every FP64 operation on the latency path is an explicit round-to-nearest
// intrinsic (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn), which nvcc never
// contracts into DFMA; the library is also built with -fmad=false.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pm2l_internal.h"

namespace pm2l {
namespace dev {

constexpr uint64_t kAbsMask = 0x7FFFFFFFFFFFFFFFull;
constexpr long long kQuietNaN = 0x7FF8000000000000ll;  // the reference's NAN bits
constexpr int kThreads = 256;

__device__ __forceinline__ double qnan() { return __longlong_as_double(kQuietNaN); }

// |x| as ordered integer bits (for x finite, compare == double compare)
__device__ __forceinline__ uint64_t abs_bits(double x) {
  return static_cast<uint64_t>(__double_as_longlong(x)) & kAbsMask;
}

__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// byte order reversal of a 64-bit word (the store's big-endian fields)
__device__ __forceinline__ uint64_t bswap64_ext(uint64_t v) {
  const uint32_t lo = uint32_t(v), hi = uint32_t(v >> 32);
  return (uint64_t(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
}

// (a + b - 1) / b in u64 exactly as the Cython kernel writes it
// (_kernels.pyx:124,126,127); 32-bit hardware path when both operands fit.
__device__ __forceinline__ uint64_t ceil_div(uint64_t a, uint64_t b) {
  const uint64_t num = a + b - 1;
  if ((num | b) <= 0xFFFFFFFFull) return uint64_t(uint32_t(num) / uint32_t(b));
  return num / b;
}

// The rare u64 division slow path kept out of line: the fully unrolled
// emission loops reach it, and inlining one u64 division per call site grows
// the lookup kernel past the instruction cache (C3 profile: "no instruction"
// stalls dominated at 130 KB of code).  Same integer result.
static __device__ __noinline__ uint64_t udiv_slow(uint64_t a, uint64_t b) { return a / b; }

// ceil((a) / d) for the curve's divisor j (0 tile_m, 1 tile_n, 2 blocks per
// wave) through the host-computed u32 magic when a + d - 1 fits in 32 bits;
// identical integer result to ceil_div.
__device__ __forceinline__ uint64_t ceil_div_c(const TablesDev& t, int c, int j, uint64_t a,
                                               uint64_t d) {
  const uint64_t num = a + d - 1;
  const uint32_t s = t.dv_s[3 * c + j];
  if ((s >> 16) && num <= 0xFFFFFFFFull) {
    const uint32_t n32 = uint32_t(num);
    const uint32_t q = __umulhi(t.dv_m[3 * c + j], n32);
    return uint64_t((q + ((n32 - q) >> (s & 0xFF))) >> ((s >> 8) & 0xFF));
  }
  return udiv_slow(num, d);
}

// compute._interpolate_detail / _kernels._interp over samples [lo, hi):
// clamp outside the sampled range, exact at samples, linear between
// neighbours: t = (k - k1) / (k3 - k1); thr = t1 + t * (t3 - t1)  (no FMA).
__device__ __forceinline__ double interp_samples(const double* __restrict__ d,
                                                 const double* __restrict__ y, int lo, int hi,
                                                 double nd) {
  if (nd < d[lo]) return y[lo];
  if (nd > d[hi - 1]) return y[hi - 1];
  int left = lo, right = hi;
  while (left < right) {
    const int mid = (left + right) >> 1;
    if (d[mid] < nd) left = mid + 1; else right = mid;
  }
  if (d[left] == nd) return y[left];
  const double k1 = d[left - 1], k3 = d[left], t1 = y[left - 1], t3 = y[left];
  const double tt = __ddiv_rn(__dsub_rn(nd, k1), __dsub_rn(k3, k1));
  return __dadd_rn(t1, __dmul_rn(tt, __dsub_rn(t3, t1)));
}

__device__ __forceinline__ double interp_thr(const TablesDev& t, int c, double nd) {
  return interp_samples(t.s_dims, t.s_thrs, t.s_off[c], t.s_off[c + 1], nd);
}

// compute._rescale first factor — depends on (curve, k) only:
// base = (ref_dur * (k / ref_dim)) * (ref_thr / thr(k))   (left-associative)
__device__ __forceinline__ double base_from_thr(const TablesDev& t, int c, double nd, double thr) {
  return __dmul_rn(__dmul_rn(t.ref_dur[c], __ddiv_rn(nd, t.ref_dim[c])),
                   __ddiv_rn(t.ref_thr[c], thr));
}

__device__ __forceinline__ double base_of(const TablesDev& t, int c, uint64_t k) {
  const double nd = __ull2double_rn(k);
  return base_from_thr(t, c, nd, interp_thr(t, c, nd));
}

// compute.block_count (78-99) in u64 (Cython semantics, _kernels.pyx:123-126).
__device__ __forceinline__ uint64_t blocks_of(const TablesDev& t, int c, uint64_t b, uint64_t m,
                                              uint64_t n, uint64_t k) {
  const uint64_t tm = t.tile_m[c];
  if (t.rowblock[c]) return ceil_div_c(t, c, 0, b * k, tm);
  return b * ceil_div_c(t, c, 0, m, tm) * ceil_div_c(t, c, 1, n, t.tile_n[c]) * t.split_k[c];
}

// waves / ref_waves  (compute.py:137, _kernels.pyx:132)
__device__ __forceinline__ double wave_scale(const TablesDev& t, int c, uint64_t waves) {
  const double w = __ull2double_rn(waves), rw = t.ref_waves[c];
  if (__builtin_expect(rw == 1.0, 1)) return w;  // x / 1.0 == x exactly (IEEE)
  return __ddiv_rn(w, rw);
}

// ceil(a / d) for a curve's divisor j (0 tile_m, 1 tile_n, 2 blocks per
// wave) from its parameters held in registers (same result as ceil_div_c)
__device__ __forceinline__ uint64_t ceil_div_p(const WcParam& p, int j, uint64_t a, uint64_t d) {
  const uint64_t num = a + d - 1;
  const uint32_t s = p.ds[j];
  if ((s >> 16) && num <= 0xFFFFFFFFull) {
    const uint32_t n32 = uint32_t(num);
    const uint32_t q = __umulhi(p.dm[j], n32);
    return uint64_t((q + ((n32 - q) >> (s & 0xFF))) >> ((s >> 8) & 0xFF));
  }
  return udiv_slow(num, d);
}

__device__ __forceinline__ WcParam curve_params(const TablesDev& t, int c) {
  WcParam q;
  q.tm = t.tile_m[c]; q.tn = t.tile_n[c]; q.sk = t.split_k[c]; q.bpw = t.bpw[c];
  q.rw = t.ref_waves[c];
#pragma unroll
  for (int j = 0; j < 3; ++j) { q.dm[j] = t.dv_m[3 * c + j]; q.ds[j] = t.dv_s[3 * c + j]; }
  return q;
}

struct PointResult {
  double lat;
  uint64_t blocks, waves;
};

// Full canonical per-point arithmetic for a known curve and its base.
__device__ __forceinline__ PointResult predict_point(const TablesDev& t, int c, uint64_t b,
                                                     uint64_t m, uint64_t n, uint64_t k,
                                                     double base) {
  PointResult r;
  r.blocks = blocks_of(t, c, b, m, n, k);
  r.waves = ceil_div_c(t, c, 2, r.blocks, t.bpw[c]);
  r.lat = __dmul_rn(base, wave_scale(t, c, r.waves));
  return r;
}

// predict_point from a curve's parameters in registers (rowblock flag apart)
__device__ __forceinline__ PointResult predict_point_p(const WcParam& p, bool rowblock, uint64_t b,
                                                       uint64_t m, uint64_t n, uint64_t k,
                                                       double base) {
  PointResult r;
  r.blocks = rowblock ? ceil_div_p(p, 0, b * k, p.tm)
                      : b * ceil_div_p(p, 0, m, p.tm) * ceil_div_p(p, 1, n, p.tn) * p.sk;
  r.waves = ceil_div_p(p, 2, r.blocks, p.bpw);
  const double w = __ull2double_rn(r.waves);
  r.lat = __dmul_rn(base, p.rw == 1.0 ? w : __ddiv_rn(w, p.rw));
  return r;
}

__device__ __forceinline__ bool curve_valid(const TablesDev& t, int c) {
  return t.s_off[c + 1] > t.s_off[c];
}

}  // namespace dev
}  // namespace pm2l
