// Memory-bound op model and per-model totals.
//   membound_kernel      predict_membound (pm2lat/membound.py:117-127): 5-feature
//                        linear model as a left-to-right FMA chain (the order
//                        OpenBLAS ddot realises behind np.dot), + intercept,
//                        floored at the launch time
//   segment_fsum_kernel  math.fsum per model (aggregate.py:193): exact
//                        warp-segmented fixed-point reduction, one warp per model
#include <algorithm>

#include "common.cuh"

namespace pm2l {
namespace {

using namespace dev;

// --------------------------------------------------------------- membound
__global__ void membound_kernel(const double* __restrict__ f, const int32_t* __restrict__ mid,
                                int64_t n, const double* __restrict__ w,
                                const double* __restrict__ icpt, const double* __restrict__ floors,
                                int64_t n_models, double* __restrict__ out,
                                uint8_t* __restrict__ floored, double* __restrict__ out_raw) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int mi = mid[i];
    if (mi < 0 || mi >= n_models) {
      out[i] = qnan();
      if (floored) floored[i] = 0;
      if (out_raw) out_raw[i] = qnan();
      continue;
    }
    const double* x = f + 5 * i;
    const double* wm = w + 5 * mi;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 5; ++j) s = __fma_rn(wm[j], x[j], s);
    const double raw = __dadd_rn(s, icpt[mi]);
    const double fl = floors[mi];
    const bool below = raw < fl;
    out[i] = below ? fl : raw;
    if (floored) floored[i] = below ? 1 : 0;
    if (out_raw) out_raw[i] = raw;
  }
}

// ------------------------------------------------------------ exact fsum
// One warp per segment.  Pass 1: max exponent E (and NaN / inf screening).
// Pass 2: every term whose bits all lie within a 4x64-bit window anchored at
// E is added or subtracted EXACTLY as a two's-complement fixed-point integer
// (integer adds are associative, so the warp tree reduction is exact); the
// 256-bit total is then rounded to nearest-even once, by magnitude, with its
// sign.  Terms are < 2^233 in window units, so |sum| < 2^255 for segments
// below 2^22 terms; longer segments and segments with a term below the
// window (dynamic range > ~180 bits) take a sequential exact expansion sum
// (Shewchuk, the algorithm behind math.fsum) on lane 0.  Signed terms are
// allowed: a raw membound layer below a non-positive floor is negative.
struct U256 {
  uint64_t w[4];
};

__device__ __forceinline__ void add256(U256& a, const U256& b) {
  asm("add.cc.u64 %0, %0, %4;\n\taddc.cc.u64 %1, %1, %5;\n\t"
      "addc.cc.u64 %2, %2, %6;\n\taddc.u64 %3, %3, %7;"
      : "+l"(a.w[0]), "+l"(a.w[1]), "+l"(a.w[2]), "+l"(a.w[3])
      : "l"(b.w[0]), "l"(b.w[1]), "l"(b.w[2]), "l"(b.w[3]));
}

__device__ __forceinline__ void sub256(U256& a, const U256& b) {
  asm("sub.cc.u64 %0, %0, %4;\n\tsubc.cc.u64 %1, %1, %5;\n\t"
      "subc.cc.u64 %2, %2, %6;\n\tsubc.u64 %3, %3, %7;"
      : "+l"(a.w[0]), "+l"(a.w[1]), "+l"(a.w[2]), "+l"(a.w[3])
      : "l"(b.w[0]), "l"(b.w[1]), "l"(b.w[2]), "l"(b.w[3]));
}

__device__ double two_sum_fsum(const double* v, int64_t lo, int64_t hi) {
  // Shewchuk/msum (the algorithm behind math.fsum), partials kept in a
  // bounded local array; exact for finite inputs of either sign.
  double p[64];
  int np = 0;
  for (int64_t i = lo; i < hi; ++i) {
    double x = v[i];
    int j = 0;
    for (int q = 0; q < np; ++q) {
      double y = p[q];
      if (fabs(x) < fabs(y)) { double tmp = x; x = y; y = tmp; }
      const double hi_ = __dadd_rn(x, y);
      const double lo_ = __dsub_rn(y, __dsub_rn(hi_, x));
      if (lo_ != 0.0) p[j++] = lo_;
      x = hi_;
    }
    if (j < 64) p[j++] = x;
    np = j;
  }
  // sum partials from the top with the half-way correction of math.fsum
  if (np == 0) return 0.0;
  double hi_ = p[--np], lo_ = 0.0;
  while (np > 0) {
    const double x = hi_, y = p[--np];
    hi_ = __dadd_rn(x, y);
    const double yr = __dsub_rn(hi_, x);
    lo_ = __dsub_rn(y, yr);
    if (lo_ != 0.0) break;
  }
  if (np > 0 && ((lo_ < 0.0 && p[np - 1] < 0.0) || (lo_ > 0.0 && p[np - 1] > 0.0))) {
    const double y = __dmul_rn(lo_, 2.0);
    const double x = __dadd_rn(hi_, y);
    const double yr = __dsub_rn(x, hi_);
    if (y == yr) hi_ = x;
  }
  return hi_ == 0.0 ? 0.0 : hi_;  // fsum of zeros is +0.0
}

__global__ void segment_fsum_kernel(const double* __restrict__ v, const int64_t* __restrict__ off,
                                    int64_t nseg, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t seg = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (seg >= nseg) return;
  const int64_t lo = off[seg], hi = off[seg + 1];
  int emax = -2000;
  bool bad_nan = false, pos_inf = false, neg_inf = false;
  for (int64_t i = lo + lane; i < hi; i += 32) {
    const double x = v[i];
    const uint64_t bits = uint64_t(__double_as_longlong(x));
    const int e = int((bits >> 52) & 0x7FF);
    if (x != x) bad_nan = true;
    else if (e == 0x7FF) { if (bits >> 63) neg_inf = true; else pos_inf = true; }
    else if (x != 0.0) emax = max(emax, e == 0 ? 1 : e);
  }
  for (int o = 16; o; o >>= 1) emax = max(emax, __shfl_xor_sync(0xFFFFFFFFu, emax, o));
  bad_nan = __any_sync(0xFFFFFFFFu, bad_nan);
  pos_inf = __any_sync(0xFFFFFFFFu, pos_inf);
  neg_inf = __any_sync(0xFFFFFFFFu, neg_inf);
  if (bad_nan || pos_inf || neg_inf) {
    // math.fsum: NaN propagates, -inf + inf raises (NaN here), else the inf
    if (lane == 0)
      out[seg] = (bad_nan || (pos_inf && neg_inf)) ? qnan()
                 : __longlong_as_double(pos_inf ? 0x7FF0000000000000ll : (long long)0xFFF0000000000000ull);
    return;
  }
  if (emax == -2000) {  // empty or all zeros
    if (lane == 0) out[seg] = 0.0;
    return;
  }
  // window: LSB weight 2^(emax - 1075 - 180); term with biased exponent e
  // (e==0 -> subnormal, scale as e=1) contributes mant << (e - emax + 180).
  constexpr int kGuard = 180;
  U256 acc = {{0, 0, 0, 0}};
  bool below = hi - lo >= (int64_t(1) << 22);
  for (int64_t i = lo + lane; i < hi && !below; i += 32) {
    const uint64_t bits = uint64_t(__double_as_longlong(v[i]));
    if ((bits << 1) == 0) continue;  // +-0
    const int be = int((bits >> 52) & 0x7FF);
    const uint64_t mant = (bits & 0xFFFFFFFFFFFFFull) | (be ? (1ull << 52) : 0ull);
    const int e = be ? be : 1;
    const int sh = e - emax + kGuard;
    if (sh < 0) { below = true; continue; }
    U256 term = {{0, 0, 0, 0}};
    const int limb = sh >> 6, bit = sh & 63;
    term.w[limb] = mant << bit;
    if (bit && limb + 1 < 4) term.w[limb + 1] = mant >> (64 - bit);
    if (bits >> 63) sub256(acc, term);
    else add256(acc, term);
  }
  below = __any_sync(0xFFFFFFFFu, below);
  if (below) {
    if (lane == 0) out[seg] = two_sum_fsum(v, lo, hi);
    return;
  }
  for (int o = 16; o; o >>= 1) {
    U256 other;
    for (int q = 0; q < 4; ++q) other.w[q] = __shfl_xor_sync(0xFFFFFFFFu, acc.w[q], o);
    add256(acc, other);
  }
  if (lane != 0) return;
  // sign and magnitude of the exact two's-complement total
  const bool negative = (acc.w[3] >> 63) != 0;
  if (negative) {
    U256 zero = {{0, 0, 0, 0}};
    sub256(zero, acc);
    acc = zero;
  }
  // round the exact 256-bit magnitude to 53 bits, nearest-even
  int top = 255;
  while (top >= 0 && !((acc.w[top >> 6] >> (top & 63)) & 1ull)) --top;
  if (top < 0) {  // exact cancellation: fsum returns +0.0
    out[seg] = 0.0;
    return;
  }
  auto bit_at = [&](int p) -> uint64_t { return p < 0 ? 0 : (acc.w[p >> 6] >> (p & 63)) & 1ull; };
  uint64_t mant = 0;
  int shift = 0;  // value = mant * 2^shift * LSB
  if (top < 53) {
    mant = acc.w[0];  // fewer than 54 significant bits: exact
  } else {
    for (int p = top; p > top - 53; --p) mant = (mant << 1) | bit_at(p);
    shift = top - 52;
    const uint64_t guard = bit_at(top - 53);
    bool sticky = false;
    for (int w = 0; w < 4 && !sticky; ++w) {
      const int lo_bit = w * 64, hi_bit = min(w * 64 + 63, top - 54);
      if (hi_bit < lo_bit) break;
      const int nbits = hi_bit - lo_bit + 1;
      const uint64_t msk = nbits >= 64 ? ~0ull : ((1ull << nbits) - 1ull);
      sticky = (acc.w[w] & msk) != 0;
    }
    if (guard && (sticky || (mant & 1ull))) {
      mant += 1;
      if (mant >> 53) { mant >>= 1; shift += 1; }
    }
  }
  // LSB weight exponent: (emax - 1075) - kGuard  (unbiased exponent of 1 ulp
  // at biased exponent emax is emax - 1075)
  const int exp2 = shift + (emax - 1075) - kGuard;
  const double mag = scalbn(double(mant), exp2);
  out[seg] = negative ? -mag : mag;
}

}  // namespace

int launch_membound(const double* f, const int32_t* mid, int64_t n, const double* w,
                    const double* b, const double* floors, int64_t n_models, double* out,
                    uint8_t* floored, double* out_raw, void* stream) {
  if (n == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = int(std::min<int64_t>((n + kThreads - 1) / kThreads, int64_t(sm_count()) * 16));
  membound_kernel<<<nb, kThreads, 0, s>>>(f, mid, n, w, b, floors, n_models, out, floored,
                                          out_raw);
  return int(cudaGetLastError());
}

int launch_segment_fsum(const double* v, const int64_t* off, int64_t nseg, double* out,
                        void* stream) {
  if (nseg == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t threads = nseg * 32;
  const int nb = int((threads + 255) / 256);
  segment_fsum_kernel<<<nb, 256, 0, s>>>(v, off, nseg, out);
  return int(cudaGetLastError());
}

}  // namespace pm2l
