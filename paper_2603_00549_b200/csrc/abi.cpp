// C entry points (include/pm2l.h): handle management, per-call staging,
// device selection, and the reference-FFI drop-in pm2l_predict_grid_slice.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <memory>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <immintrin.h>
#include <mutex>
#include <string>
#include <unordered_map>
#include <thread>

#include <nvtx3/nvToolsExt.h>
#include <vector>

#include "../../include/pm2l.h"
#include "pm2l_internal.h"

using namespace pm2l;

namespace {

thread_local std::string g_error;

// NVTX range over one C-ABI call (header-only NVTX v3: a no-op unless a
// profiler such as nsys / ncu --nvtx is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(PM2L_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                                 cudaGetErrorString(e) + ")");
}

#define PM2L_CUDA(call)                                   \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);   \
  } while (0)

// Growable device / pinned host buffers.
struct DeviceBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t want = std::max(need, size_t(4096));
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

struct PinnedBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    size_t want = std::max(need, size_t(4096));
    cudaError_t e = cudaMallocHost(&ptr, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

int check_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(PM2L_ERR_NODEVICE,
                "no CUDA device visible: the B200 build has no CPU fallback");
  return PM2L_OK;
}

// libm log2 of every integer below kLutN, per device (explicit-descriptor mode).
constexpr int64_t kLutN = int64_t(1) << 22;
std::mutex g_lut_mu;
std::unordered_map<int, double*> g_lut;

int get_lut(int device, double** out) {
  std::lock_guard<std::mutex> lk(g_lut_mu);
  auto it = g_lut.find(device);
  if (it != g_lut.end()) {
    *out = it->second;
    return PM2L_OK;
  }
  std::vector<double> host(kLutN);
  host[0] = -INFINITY;
  for (int64_t v = 1; v < kLutN; ++v) host[v] = std::log2(double(v));
  double* d = nullptr;
  PM2L_CUDA(cudaMalloc(&d, kLutN * sizeof(double)));
  PM2L_CUDA(cudaMemcpy(d, host.data(), kLutN * sizeof(double), cudaMemcpyHostToDevice));
  PM2L_CUDA(cudaDeviceSynchronize());  // complete before any stream may read it
  g_lut[device] = d;
  *out = d;
  return PM2L_OK;
}

}  // namespace

namespace pm2l {
int sm_count() {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  cache[dev] = n;
  return n;
}
}  // namespace pm2l

struct pm2l_grid_dplan {
  pm2l_tables* tables = nullptr;
  DPlanCaps caps;
  DeviceBuf buf;        // plan arrays + axis slots
  DeviceBuf workspace;  // base table [C x max_k]
  GridDev last{};       // the last launched slice (diagnostics)
  int path = -1;        // grid kernel of the last launch
};

struct pm2l_tables {
  int device = 0;
  TablesHost host;
  TablesDev dev;
  DeviceBuf blob;
  // host-axis calls on canonical axes plan on the device (grown on demand)
  std::unique_ptr<pm2l_grid_dplan> hplan;
  PinnedBuf axes_pinned;
  // per-call staging (guarded by mu; reused once the previous call's work
  // has drained, tracked by `done`)
  std::mutex mu;
  PinnedBuf grid_pinned;
  DeviceBuf grid_dev;
  DeviceBuf workspace;
  cudaEvent_t done = nullptr;
  bool pending = false;
};

namespace {

// Axes the device planner takes: strictly ascending, values in [1, kLutN).
bool canonical_axes(const uint64_t* const axes[4], const int64_t lens[4]) {
  for (int a = 0; a < 4; ++a) {
    if (lens[a] < 1 || !axes[a]) return false;
    for (int64_t i = 0; i < lens[a]; ++i) {
      const uint64_t v = axes[a][i];
      if (v == 0 || (a > 0 && v >= uint64_t(kLutN)) || (i > 0 && !(axes[a][i - 1] < v)))
        return false;
    }
  }
  return true;
}

int dplan_reserve(pm2l_grid_dplan* p, const DPlanCaps& need) {
  DPlanCaps c = p->caps;
  if (need.nB <= c.nB && need.nM <= c.nM && need.nN <= c.nN && need.nK <= c.nK && p->buf.ptr)
    return PM2L_OK;
  c.nB = std::max(c.nB, need.nB); c.nM = std::max(c.nM, need.nM);
  c.nN = std::max(c.nN, need.nN); c.nK = std::max(c.nK, need.nK);
  const TablesDev& t = p->tables->dev;
  if (!dplan_supported(t, c)) return fail(PM2L_ERR_INVALID, "slice too large for the device planner");
  p->buf.release();
  PM2L_CUDA(p->buf.reserve(size_t(dplan_bytes(t, c))));
  PM2L_CUDA(cudaMemset(p->buf.ptr, 0, size_t(dplan_bytes(t, c))));
  // cudaMemset runs on the legacy default stream, which the callers'
  // non-blocking streams do not order against: without this wait the zero
  // fill could land after (and erase) the first call's axis upload
  PM2L_CUDA(cudaDeviceSynchronize());
  PM2L_CUDA(p->workspace.reserve(size_t(std::max<int64_t>(int64_t(t.C) * c.nK, 1)) * sizeof(double)));
  p->caps = c;
  return PM2L_OK;
}

// GridDev of a device-planned slice (device axis pointers, or the plan's own
// axis slots when axes[a] is null).
int dplan_grid_for(pm2l_grid_dplan* p, const uint64_t* const axes[4], const int64_t lens[4],
                   int64_t b_lo, int64_t b_hi, GridDev* g) {
  for (int a = 0; a < 4; ++a)
    if (lens[a] < 1) return fail(PM2L_ERR_INVALID, "device-planned axes must be non-empty");
  if (b_lo < 0 || b_hi < b_lo || b_hi > lens[0]) return fail(PM2L_ERR_INVALID, "batch slice out of range");
  if (lens[0] > p->caps.nB || lens[1] > p->caps.nM || lens[2] > p->caps.nN || lens[3] > p->caps.nK)
    return fail(PM2L_ERR_INVALID, "axes exceed the device plan's capacity");
  double* lut = nullptr;
  if (int rc = get_lut(p->tables->device, &lut)) return rc;
  *g = dplan_grid(p->tables->dev, p->caps, p->buf.ptr, axes, lens, b_lo, b_hi);
  g->lut = lut;
  g->lut_n = kLutN;
  return PM2L_OK;
}

int stage_grid(pm2l_tables* t, const uint64_t* const axes[4], const int64_t lens[4],
               int64_t b_lo, int64_t b_hi, cudaStream_t s, GridDev* g) {
  if (t->pending) {
    PM2L_CUDA(cudaEventSynchronize(t->done));
    t->pending = false;
  }
  const DPlanCaps need{lens[0], lens[1], lens[2], lens[3]};
  if (b_lo >= 0 && b_hi >= b_lo && b_hi <= lens[0] && dplan_supported(t->dev, need) &&
      canonical_axes(axes, lens)) {
    // canonical axes: upload them (a few KB) and plan on the device
    if (!t->hplan) {
      t->hplan.reset(new pm2l_grid_dplan());
      t->hplan->tables = t;
    }
    pm2l_grid_dplan* p = t->hplan.get();
    if (int rc = dplan_reserve(p, need)) return rc;
    size_t bytes = 0;
    for (int a = 0; a < 4; ++a) bytes += size_t(lens[a]) * 8;
    PM2L_CUDA(t->axes_pinned.reserve(bytes));
    uint8_t* hp = static_cast<uint8_t*>(t->axes_pinned.ptr);
    for (int a = 0; a < 4; ++a) {
      std::memcpy(hp, axes[a], size_t(lens[a]) * 8);
      PM2L_CUDA(cudaMemcpyAsync(dplan_axis_slot(t->dev, p->caps, p->buf.ptr, a), hp,
                                size_t(lens[a]) * 8, cudaMemcpyHostToDevice, s));
      hp += size_t(lens[a]) * 8;
    }
    const uint64_t* none[4] = {nullptr, nullptr, nullptr, nullptr};
    return dplan_grid_for(p, none, lens, b_lo, b_hi, g);
  }
  GridHost gh;
  std::string err = build_grid(t->host, axes, lens, b_lo, b_hi, &gh);
  if (!err.empty()) return fail(PM2L_ERR_INVALID, err);
  PM2L_CUDA(t->grid_pinned.reserve(gh.blob.size()));
  PM2L_CUDA(t->grid_dev.reserve(gh.blob.size()));
  std::memcpy(t->grid_pinned.ptr, gh.blob.data(), gh.blob.size());
  PM2L_CUDA(cudaMemcpyAsync(t->grid_dev.ptr, t->grid_pinned.ptr, gh.blob.size(),
                            cudaMemcpyHostToDevice, s));
  *g = rebase(gh.dev_offsets, t->grid_dev.ptr);
  return PM2L_OK;
}

int finish_call(pm2l_tables* t, cudaStream_t s) {
  PM2L_CUDA(cudaEventRecord(t->done, s));
  t->pending = true;
  return PM2L_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int pm2l_abi_version(void) { return PM2L_ABI_VERSION; }

#ifndef PM2L_SOURCE_HASH
#define PM2L_SOURCE_HASH "unknown"
#endif
const char* pm2l_source_hash(void) { return PM2L_SOURCE_HASH; }

const char* pm2l_last_error(void) { return g_error.c_str(); }

int pm2l_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int pm2l_tables_create(const pm2l_tables_view* view, int device, pm2l_tables** out) {
  NvtxRange nvtx_("pm2l_tables_create");
  if (!out) return fail(PM2L_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (int rc = check_device()) return rc;
  std::unique_ptr<pm2l_tables> t(new pm2l_tables());
  t->device = device;
  std::string err = build_tables(view, &t->host);
  if (!err.empty()) return fail(PM2L_ERR_INVALID, err);
  DeviceGuard guard(device);
  PM2L_CUDA(t->blob.reserve(std::max<size_t>(t->host.blob.size(), 256)));
  if (!t->host.blob.empty())
    PM2L_CUDA(cudaMemcpy(t->blob.ptr, t->host.blob.data(), t->host.blob.size(),
                         cudaMemcpyHostToDevice));
  // a pageable-source cudaMemcpy may return before its DMA lands, and
  // launches on non-blocking streams (the drop-in's) are not ordered after
  // it: the tables must be complete before the handle is handed out
  PM2L_CUDA(cudaDeviceSynchronize());
  t->dev = rebase(t->host.dev_offsets, t->blob.ptr);
  PM2L_CUDA(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming));
  *out = t.release();
  return PM2L_OK;
}

int pm2l_tables_destroy(pm2l_tables* t) {
  if (!t) return PM2L_OK;
  {
    DeviceGuard guard(t->device);
    if (t->pending) cudaEventSynchronize(t->done);
    if (t->done) cudaEventDestroy(t->done);
    t->blob.release();
    t->grid_dev.release();
    t->workspace.release();
    t->grid_pinned.release();
    t->axes_pinned.release();
    if (t->hplan) {
      t->hplan->buf.release();
      t->hplan->workspace.release();
    }
  }
  delete t;
  return PM2L_OK;
}

int64_t pm2l_tables_groups(const pm2l_tables* t) { return t ? t->dev.G : -1; }

int pm2l_grid_predict(pm2l_tables* t, const uint64_t* batch_vals, int64_t n_batch,
                      const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals, int64_t n_n,
                      const uint64_t* k_vals, int64_t n_k, int64_t b_lo, int64_t b_hi,
                      double* out_lat, int32_t* out_curve, uint64_t* out_blocks,
                      uint64_t* out_waves, void* stream) {
  NvtxRange nvtx_("pm2l_grid_predict");
  if (!t) return fail(PM2L_ERR_INVALID, "null tables");
  const bool any_v = out_curve || out_blocks || out_waves;
  if (any_v && !(out_curve && out_blocks && out_waves))
    return fail(PM2L_ERR_INVALID, "out_curve/out_blocks/out_waves must be all set or all NULL");
  std::lock_guard<std::mutex> lk(t->mu);
  DeviceGuard guard(t->device);
  const uint64_t* axes[4] = {batch_vals, m_vals, n_vals, k_vals};
  const int64_t lens[4] = {n_batch, n_m, n_n, n_k};
  if (n_m * n_n * n_k * (b_hi - b_lo) > 0 && !out_lat)
    return fail(PM2L_ERR_INVALID, "null out_lat");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GridDev g;
  if (int rc = stage_grid(t, axes, lens, b_lo, b_hi, s, &g)) return rc;
  const int64_t ws = grid_workspace_elems(t->dev, g);
  if (ws > 0) PM2L_CUDA(t->workspace.reserve(size_t(ws) * sizeof(double)));
  LaunchOut o{out_lat, out_curve, out_blocks, out_waves};
  const int rc = launch_grid(t->dev, g, t->host.max_group,
                             ws > 0 ? static_cast<double*>(t->workspace.ptr) : nullptr, ws, o, s);
  if (g.dev_planned) t->hplan->path = grid_kernel_path(t->dev, g, o);
  if (rc) return cuda_fail(cudaError_t(rc), "grid kernel launch");
  return finish_call(t, s);
}

struct pm2l_grid_plan {
  pm2l_tables* tables = nullptr;
  GridDev grid;
  DeviceBuf blob;
  DeviceBuf workspace;
  int64_t ws_elems = 0;
  int64_t staged_bytes = 0;
};

int pm2l_grid_plan_create(pm2l_tables* t, const uint64_t* batch_vals, int64_t n_batch,
                          const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals,
                          int64_t n_n, const uint64_t* k_vals, int64_t n_k, int64_t b_lo,
                          int64_t b_hi, pm2l_grid_plan** out) {
  NvtxRange nvtx_("pm2l_grid_plan_create");
  if (!t || !out) return fail(PM2L_ERR_INVALID, "null tables/output handle");
  *out = nullptr;
  DeviceGuard guard(t->device);
  const uint64_t* axes[4] = {batch_vals, m_vals, n_vals, k_vals};
  const int64_t lens[4] = {n_batch, n_m, n_n, n_k};
  GridHost gh;
  std::string err = build_grid(t->host, axes, lens, b_lo, b_hi, &gh);
  if (!err.empty()) return fail(PM2L_ERR_INVALID, err);
  std::unique_ptr<pm2l_grid_plan> p(new pm2l_grid_plan());
  p->tables = t;
  PM2L_CUDA(p->blob.reserve(gh.blob.size()));
  PM2L_CUDA(cudaMemcpy(p->blob.ptr, gh.blob.data(), gh.blob.size(), cudaMemcpyHostToDevice));
  PM2L_CUDA(cudaDeviceSynchronize());  // the plan is complete before any stream may read it
  p->grid = rebase(gh.dev_offsets, p->blob.ptr);
  p->staged_bytes = int64_t(gh.blob.size());
  p->ws_elems = grid_workspace_elems(t->dev, p->grid);
  if (p->ws_elems > 0) PM2L_CUDA(p->workspace.reserve(size_t(p->ws_elems) * sizeof(double)));
  *out = p.release();
  return PM2L_OK;
}

int pm2l_grid_plan_launch(pm2l_grid_plan* p, double* out_lat, int32_t* out_curve,
                          uint64_t* out_blocks, uint64_t* out_waves, uint64_t* nan_stats,
                          int stages, void* stream) {
  NvtxRange nvtx_("pm2l_grid_plan_launch");
  if (!p) return fail(PM2L_ERR_INVALID, "null plan");
  const bool any_v = out_curve || out_blocks || out_waves;
  if (any_v && !(out_curve && out_blocks && out_waves))
    return fail(PM2L_ERR_INVALID, "out_curve/out_blocks/out_waves must be all set or all NULL");
  const GridDev& g = p->grid;
  if ((g.b_hi - g.b_lo) * g.nM * g.nN * g.nK > 0 && !out_lat)
    return fail(PM2L_ERR_INVALID, "null out_lat");
  DeviceGuard guard(p->tables->device);
  LaunchOut o{out_lat, out_curve, out_blocks, out_waves,
              reinterpret_cast<unsigned long long*>(nan_stats)};
  const int rc = launch_grid(p->tables->dev, g, p->tables->host.max_group,
                             p->ws_elems > 0 ? static_cast<double*>(p->workspace.ptr) : nullptr,
                             p->ws_elems, o, stream, stages ? stages : kStageAll);
  if (rc) return cuda_fail(cudaError_t(rc), "grid plan launch");
  return PM2L_OK;
}

int pm2l_grid_plan_info(const pm2l_grid_plan* p, int64_t* info) {
  if (!p || !info) return fail(PM2L_ERR_INVALID, "null plan/info");
  const GridDev& g = p->grid;
  info[0] = (g.b_hi - g.b_lo) * g.nM * g.nN * g.nK;
  info[1] = g.n_fix;
  info[2] = p->ws_elems * int64_t(sizeof(double));
  info[3] = p->staged_bytes;
  return PM2L_OK;
}

int pm2l_grid_plan_kernel(const pm2l_grid_plan* p, const double* out_lat, int verify) {
  if (!p) return fail(PM2L_ERR_INVALID, "null plan");
  int32_t dummy = 0;
  LaunchOut o{const_cast<double*>(out_lat), verify ? &dummy : nullptr};
  return grid_kernel_path(p->tables->dev, p->grid, o);
}

#ifdef PM2L_TIMING
int pm2l_debug_row_timing(unsigned long long* host, int n) {
  return pm2l::row_timing_copy(host, n);
}
int pm2l_debug_plan_timing(unsigned long long* host, int n) {
  if (!pm2l::plan_timing_buffer()) return -1;
  return int(cudaMemcpy(host, pm2l::plan_timing_buffer(), sizeof(unsigned long long) * size_t(n),
                        cudaMemcpyDeviceToHost));
}
#endif

int pm2l_grid_plan_destroy(pm2l_grid_plan* p) {
  if (!p) return PM2L_OK;
  {
    DeviceGuard guard(p->tables->device);
    cudaDeviceSynchronize();
    p->blob.release();
    p->workspace.release();
  }
  delete p;
  return PM2L_OK;
}

int pm2l_grid_dplan_create(pm2l_tables* t, int64_t max_batch, int64_t max_m, int64_t max_n,
                           int64_t max_k, pm2l_grid_dplan** out) {
  if (!t || !out) return fail(PM2L_ERR_INVALID, "null tables/output handle");
  *out = nullptr;
  if (max_batch < 1 || max_m < 1 || max_n < 1 || max_k < 1)
    return fail(PM2L_ERR_INVALID, "device plan capacities must be >= 1");
  DeviceGuard guard(t->device);
  std::unique_ptr<pm2l_grid_dplan> p(new pm2l_grid_dplan());
  p->tables = t;
  if (!dplan_supported(t->dev, DPlanCaps{max_batch, max_m, max_n, max_k}))
    return fail(PM2L_ERR_INVALID, "tables or capacities outside the device planner's range");
  if (int rc = dplan_reserve(p.get(), DPlanCaps{max_batch, max_m, max_n, max_k})) return rc;
  double* lut = nullptr;
  if (int rc = get_lut(t->device, &lut)) return rc;  // built once per device, before any capture
  *out = p.release();
  return PM2L_OK;
}

int pm2l_grid_dplan_launch(pm2l_grid_dplan* p, const uint64_t* batch_vals, int64_t n_batch,
                           const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals,
                           int64_t n_n, const uint64_t* k_vals, int64_t n_k, int64_t b_lo,
                           int64_t b_hi, double* out_lat, int32_t* out_curve,
                           uint64_t* out_blocks, uint64_t* out_waves, uint64_t* nan_stats,
                           int stages, void* stream) {
  NvtxRange nvtx_("pm2l_grid_dplan_launch");
  if (!p) return fail(PM2L_ERR_INVALID, "null device plan");
  const bool any_v = out_curve || out_blocks || out_waves;
  if (any_v && !(out_curve && out_blocks && out_waves))
    return fail(PM2L_ERR_INVALID, "out_curve/out_blocks/out_waves must be all set or all NULL");
  if (!batch_vals || !m_vals || !n_vals || !k_vals) return fail(PM2L_ERR_INVALID, "null axis");
  if (!out_lat) return fail(PM2L_ERR_INVALID, "null out_lat");
  DeviceGuard guard(p->tables->device);
  const uint64_t* axes[4] = {batch_vals, m_vals, n_vals, k_vals};
  const int64_t lens[4] = {n_batch, n_m, n_n, n_k};
  GridDev g;
  if (int rc = dplan_grid_for(p, axes, lens, b_lo, b_hi, &g)) return rc;
  LaunchOut o{out_lat, out_curve, out_blocks, out_waves,
              reinterpret_cast<unsigned long long*>(nan_stats)};
  const int64_t ws = grid_workspace_elems(p->tables->dev, g);
  const int rc = launch_grid(p->tables->dev, g, p->tables->host.max_group,
                             static_cast<double*>(p->workspace.ptr),
                             std::max<int64_t>(ws, int64_t(p->tables->dev.C) * p->caps.nK), o,
                             stream, stages ? stages : kStageAll);
  if (rc) return cuda_fail(cudaError_t(rc), "device-planned grid launch");
  p->last = g;
  p->path = grid_kernel_path(p->tables->dev, g, o);
  return PM2L_OK;
}

int pm2l_grid_dplan_status(pm2l_grid_dplan* p, uint32_t* status) {
  if (!p || !status) return fail(PM2L_ERR_INVALID, "null device plan/status");
  DeviceGuard guard(p->tables->device);
  const GridDev g = dplan_grid(p->tables->dev, p->caps, p->buf.ptr, nullptr,
                               std::array<int64_t, 4>{1, 1, 1, 1}.data(), 0, 1);
  PM2L_CUDA(cudaDeviceSynchronize());
  PM2L_CUDA(cudaMemcpy(status, g.status, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  PM2L_CUDA(cudaMemset(g.status, 0, sizeof(uint32_t)));
  PM2L_CUDA(cudaDeviceSynchronize());  // cleared before any non-blocking stream plans again
  return PM2L_OK;
}

int pm2l_grid_dplan_kernel(const pm2l_grid_dplan* p) {
  if (!p) return fail(PM2L_ERR_INVALID, "null device plan");
  return p->path;
}

int pm2l_grid_dplan_fixups(pm2l_grid_dplan* p, int64_t* count) {
  if (!p || !count) return fail(PM2L_ERR_INVALID, "null device plan/count");
  DeviceGuard guard(p->tables->device);
  PM2L_CUDA(cudaDeviceSynchronize());
  std::vector<int64_t> pos(size_t(std::max<int64_t>(p->last.n_fix, 0)));
  if (!pos.empty())
    PM2L_CUDA(cudaMemcpy(pos.data(), p->last.fix_pos, pos.size() * sizeof(int64_t),
                         cudaMemcpyDeviceToHost));
  *count = std::count_if(pos.begin(), pos.end(), [](int64_t v) { return v >= 0; });
  return PM2L_OK;
}

int pm2l_grid_dplan_destroy(pm2l_grid_dplan* p) {
  if (!p) return PM2L_OK;
  {
    DeviceGuard guard(p->tables->device);
    cudaDeviceSynchronize();
    p->buf.release();
    p->workspace.release();
  }
  delete p;
  return PM2L_OK;
}

int pm2l_nan_scan(const double* lat, int64_t n, uint64_t* first, void* stream) {
  NvtxRange nvtx_("pm2l_nan_scan");
  if (n < 0 || (n > 0 && (!lat || !first))) return fail(PM2L_ERR_INVALID, "bad nan_scan args");
  if (int rc = check_device()) return rc;
  const int rc = launch_nan_scan(lat, n, reinterpret_cast<unsigned long long*>(first), stream);
  if (rc) return cuda_fail(cudaError_t(rc), "nan scan launch");
  return PM2L_OK;
}

int pm2l_grid_predict_all_curves(pm2l_tables* t, const uint64_t* batch_vals, int64_t n_batch,
                                 const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals,
                                 int64_t n_n, const uint64_t* k_vals, int64_t n_k, int64_t b_lo,
                                 int64_t b_hi, double* out_lat, void* stream) {
  NvtxRange nvtx_("pm2l_grid_predict_all_curves");
  if (!t) return fail(PM2L_ERR_INVALID, "null tables");
  std::lock_guard<std::mutex> lk(t->mu);
  DeviceGuard guard(t->device);
  const uint64_t* axes[4] = {batch_vals, m_vals, n_vals, k_vals};
  const int64_t lens[4] = {n_batch, n_m, n_n, n_k};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GridDev g;
  if (int rc = stage_grid(t, axes, lens, b_lo, b_hi, s, &g)) return rc;
  const int64_t ws = int64_t(t->dev.C) * n_k;
  PM2L_CUDA(t->workspace.reserve(size_t(std::max<int64_t>(ws, 1)) * sizeof(double)));
  const int rc = launch_grid_all_curves(t->dev, g, static_cast<double*>(t->workspace.ptr),
                                        out_lat, s);
  if (rc) return cuda_fail(cudaError_t(rc), "all-curves kernel launch");
  return finish_call(t, s);
}

int pm2l_points_predict_ext(pm2l_tables* t, const uint32_t* shapes, int64_t n,
                            const uint32_t* ext_coords, const double* ext_log2, int64_t n_ext,
                            double* out_lat, int32_t* out_curve, uint32_t* out_waves,
                            int8_t* out_match, int32_t* out_record, double* out_dist,
                            double* out_detail, void* stream) {
  NvtxRange nvtx_("pm2l_points_predict_ext");
  if (!t) return fail(PM2L_ERR_INVALID, "null tables");
  if (n < 0 || n_ext < 0) return fail(PM2L_ERR_INVALID, "negative count");
  if (n > 0 && (!shapes || !out_lat)) return fail(PM2L_ERR_INVALID, "null shapes/out_lat");
  if (n_ext > 0 && (!ext_coords || !ext_log2)) return fail(PM2L_ERR_INVALID, "null log2 extension");
  if (n_ext > (int64_t(1) << 31)) return fail(PM2L_ERR_INVALID, "log2 extension too long");
  DeviceGuard guard(t->device);
  LogSource logs;
  if (int rc = get_lut(t->device, const_cast<double**>(&logs.lut))) return rc;
  logs.lut_n = kLutN;
  logs.ext_coord = ext_coords;
  logs.ext_log = ext_log2;
  logs.n_ext = n_ext;
  const int rc = launch_points(t->dev, shapes, n, logs, out_lat, out_curve, out_waves, out_match,
                               out_record, out_dist, out_detail, stream);
  if (rc) return cuda_fail(cudaError_t(rc), "points kernel launch");
  return PM2L_OK;
}

int pm2l_points_predict(pm2l_tables* t, const uint32_t* shapes, int64_t n, double* out_lat,
                        int32_t* out_curve, uint32_t* out_waves, int8_t* out_match,
                        int32_t* out_record, double* out_dist, void* stream) {
  return pm2l_points_predict_ext(t, shapes, n, nullptr, nullptr, 0, out_lat, out_curve, out_waves,
                                 out_match, out_record, out_dist, nullptr, stream);
}

int64_t pm2l_points_log2_table_size(void) { return kLutN; }

int pm2l_points_predict_curve(pm2l_tables* t, const uint32_t* shapes, const int32_t* curve_ids,
                              int64_t n, double* out_lat, uint32_t* out_waves,
                              double* out_detail, void* stream) {
  NvtxRange nvtx_("pm2l_points_predict_curve");
  if (!t) return fail(PM2L_ERR_INVALID, "null tables");
  if (n < 0) return fail(PM2L_ERR_INVALID, "negative count");
  if (n > 0 && (!shapes || !curve_ids || !out_lat))
    return fail(PM2L_ERR_INVALID, "null shapes/curve_ids/out_lat");
  DeviceGuard guard(t->device);
  const int rc = launch_points_curve(t->dev, shapes, curve_ids, n, out_lat, out_waves, out_detail,
                                     stream);
  if (rc) return cuda_fail(cudaError_t(rc), "points-curve kernel launch");
  return PM2L_OK;
}

int pm2l_membound_predict_raw(const double* features, const int32_t* model_ids, int64_t n,
                              const double* weights, const double* intercepts,
                              const double* floors, int64_t n_models, double* out_lat,
                              uint8_t* out_floored, double* out_raw, void* stream) {
  NvtxRange nvtx_("pm2l_membound_predict");
  if (n < 0 || n_models < 0) return fail(PM2L_ERR_INVALID, "negative count");
  if (n > 0 && (!features || !model_ids || !out_lat || !weights || !intercepts || !floors))
    return fail(PM2L_ERR_INVALID, "null membound argument");
  if (int rc = check_device()) return rc;
  const int rc = launch_membound(features, model_ids, n, weights, intercepts, floors, n_models,
                                 out_lat, out_floored, out_raw, stream);
  if (rc) return cuda_fail(cudaError_t(rc), "membound kernel launch");
  return PM2L_OK;
}

int pm2l_membound_predict(const double* features, const int32_t* model_ids, int64_t n,
                          const double* weights, const double* intercepts, const double* floors,
                          int64_t n_models, double* out_lat, uint8_t* out_floored, void* stream) {
  return pm2l_membound_predict_raw(features, model_ids, n, weights, intercepts, floors, n_models,
                                   out_lat, out_floored, nullptr, stream);
}

int pm2l_segment_fsum(const double* values, const int64_t* offsets, int64_t n_segments,
                      double* out_totals, void* stream) {
  NvtxRange nvtx_("pm2l_segment_fsum");
  if (n_segments < 0) return fail(PM2L_ERR_INVALID, "negative count");
  if (n_segments > 0 && (!values || !offsets || !out_totals))
    return fail(PM2L_ERR_INVALID, "null fsum argument");
  if (int rc = check_device()) return rc;
  const int rc = launch_segment_fsum(values, offsets, n_segments, out_totals, stream);
  if (rc) return cuda_fail(cudaError_t(rc), "fsum kernel launch");
  return PM2L_OK;
}

int pm2l_grid_error_report(const int64_t* dims, const double* thrs, int64_t n_samples,
                           int64_t stride, const double* truth, const int64_t* scan_off,
                           const double* rational, double* out_err, int64_t* out_argmax,
                           void* stream) {
  NvtxRange nvtx_("pm2l_grid_error_report");
  if (n_samples < 2) return fail(PM2L_ERR_INVALID, "a curve needs >= 2 samples");
  if (n_samples > 1024) return fail(PM2L_ERR_INVALID, "more than 1024 samples");
  if (stride < 1) return fail(PM2L_ERR_INVALID, "stride must be >= 1");
  if (!dims || !thrs || !out_err || !out_argmax || (!truth && !rational) || (truth && !scan_off))
    return fail(PM2L_ERR_INVALID, "null grid-error argument");
  if (int rc = check_device()) return rc;
  const int rc = launch_grid_error(dims, thrs, int(n_samples), stride, truth, scan_off, rational,
                                   out_err, out_argmax, stream);
  if (rc) return cuda_fail(cudaError_t(rc), "grid-error kernel launch");
  return PM2L_OK;
}

int pm2l_partition_scan(const double* lat_a, const double* lat_b, int64_t n_layers,
                        const double* transfer, double* out_stage_a, double* out_stage_b,
                        double* out_bottleneck, int64_t* out_best_cut, void* stream) {
  NvtxRange nvtx_("pm2l_partition_scan");
  if (n_layers < 0) return fail(PM2L_ERR_INVALID, "negative layer count");
  if ((n_layers > 0 && (!lat_a || !lat_b)) || !out_stage_a || !out_stage_b || !out_bottleneck ||
      !out_best_cut)
    return fail(PM2L_ERR_INVALID, "null partition argument");
  if (int rc = check_device()) return rc;
  const int rc = launch_partition(lat_a, lat_b, n_layers, transfer, out_stage_a, out_stage_b,
                                  out_bottleneck, out_best_cut, stream);
  if (rc) return cuda_fail(cudaError_t(rc), "partition kernel launch");
  return PM2L_OK;
}

int64_t pm2l_store_encode_workspace(int64_t n) { return n < 0 ? -1 : store_encode_workspace(n); }

int pm2l_store_encode(const double* lat, int64_t n, const uint64_t* batch_vals,
                      const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals, int64_t n_n,
                      const uint64_t* k_vals, int64_t n_k, void* workspace, uint8_t* records,
                      int64_t* count, void* stream) {
  NvtxRange nvtx_("pm2l_store_encode");
  if (n < 0 || n_m < 0 || n_n < 0 || n_k < 0) return fail(PM2L_ERR_INVALID, "negative size");
  if (!count) return fail(PM2L_ERR_INVALID, "null count");
  if (n > 0 && (!lat || !batch_vals || !m_vals || !n_vals || !k_vals || !workspace || !records))
    return fail(PM2L_ERR_INVALID, "null store_encode argument");
  if (n > 0 && n % (n_m * n_n * n_k) != 0)
    return fail(PM2L_ERR_INVALID, "n is not a whole number of batch planes");
  if (int rc = check_device()) return rc;
  const int rc = launch_store_encode(lat, n, batch_vals, m_vals, n_m, n_vals, n_n, k_vals, n_k,
                                     workspace, records, count, stream);
  if (rc) return cuda_fail(cudaError_t(rc), "store encode launch");
  return PM2L_OK;
}

int pm2l_store_lookup(const uint8_t* records, int64_t n_records, const uint64_t* const* axes,
                      const int64_t* axis_lens, const uint64_t* queries, int64_t n, double* out,
                      uint64_t* first_missing, void* stream) {
  NvtxRange nvtx_("pm2l_store_lookup");
  if (n < 0 || n_records < 0) return fail(PM2L_ERR_INVALID, "negative size");
  if (n > 0 && (!queries || !out || !first_missing || (n_records > 0 && !records)))
    return fail(PM2L_ERR_INVALID, "null store_lookup argument");
  if (int rc = check_device()) return rc;
  const uint64_t* ax[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t lens[4] = {0, 0, 0, 0};
  bool dense = axes != nullptr && axis_lens != nullptr;
  if (dense) {
    int64_t prod = 1;
    for (int a = 0; a < 4; ++a) {
      ax[a] = axes[a];
      lens[a] = axis_lens[a];
      if (!ax[a] || lens[a] < 1) dense = false;
      prod *= lens[a];
    }
    dense = dense && prod == n_records;
  }
  const int rc = launch_store_lookup(records, n_records, dense ? ax : nullptr, lens, queries, n,
                                     out, reinterpret_cast<unsigned long long*>(first_missing),
                                     stream);
  if (rc) return cuda_fail(cudaError_t(rc), "store lookup launch");
  return PM2L_OK;
}

// ------------------------------------------------------------------ drop-in
namespace {

// FNV-1a style content hash over 8-byte words (one dependent multiply per
// word instead of per byte: the tables are hashed on every call), then the
// tail bytes
uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, b + i, 8);
    h = (h ^ w) * 0x100000001b3ull;
    h ^= h >> 29;
  }
  for (; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  return h;
}

// memcpy with non-temporal stores for the destination (the caller's result
// buffer is written once and not read back here: no read-for-ownership of
// its lines, which halves the host memory traffic of the copy-out)
__attribute__((target("avx2"))) void copy_nt_avx2(uint8_t* dst, const uint8_t* src, size_t n) {
  size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head; src += head; n -= head;
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

void copy_out(void* dst, const void* src, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) copy_nt_avx2(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), n);
  else std::memcpy(dst, src, n);
}

// Persistent host worker threads for the pinned-staging -> caller-buffer
// copies of the drop-in's result (a single memcpy thread reaches a fraction
// of the host's memory bandwidth; the caller's numpy buffer is pageable).
// Workers spin briefly for the next job before sleeping, so a job costs
// microseconds to dispatch within a call and nothing between calls.
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) threads_.emplace_back([this, i] { run(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& th : threads_) th.join();
  }
  int parts() const { return int(threads_.size()) + 1; }
  // copy_out(dst, src, n) split over the workers and the calling thread
  void copy(void* dst, const void* src, size_t n) {
    const int P = parts();
    piece_ = ((n + P - 1) / P + 4095) & ~size_t(4095);
    dst_ = static_cast<uint8_t*>(dst);
    src_ = static_cast<const uint8_t*>(src);
    n_ = n;
    pending_.store(int(threads_.size()), std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    part(0);
    while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
  }

 private:
  void part(int p) {
    const size_t lo = std::min(n_, size_t(p) * piece_), hi = std::min(n_, lo + piece_);
    if (hi > lo) copy_out(dst_ + lo, src_ + lo, hi - lo);
  }
  void run(int i) {
    uint64_t seen = 0;
    for (;;) {
      // spin ~100 us for the next job, then sleep
      bool got = false;
      for (int k = 0; k < 20000 && !got; ++k) {
        if (stop_.load(std::memory_order_relaxed)) return;
        got = gen_.load(std::memory_order_acquire) != seen;
        if (!got) _mm_pause();
      }
      if (!got) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_.load() || gen_.load() != seen; });
        if (stop_.load()) return;
      }
      seen = gen_.load(std::memory_order_acquire);
      part(i + 1);
      pending_.fetch_sub(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<bool> stop_{false};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  uint8_t* dst_ = nullptr;
  const uint8_t* src_ = nullptr;
  size_t n_ = 0, piece_ = 0;
};

constexpr int kStageBufs = 4;
// bytes per D2H chunk (PM2L_STAGE_CHUNK_MB overrides it for tuning; read once)
size_t stage_chunk() {
  static const size_t v = [] {
    const char* e = std::getenv("PM2L_STAGE_CHUNK_MB");
    const long mb = e ? std::atol(e) : 0;
    return size_t(mb > 0 && mb <= 64 ? mb : 8) << 20;
  }();
  return v;
}

struct SliceDevice {
  DeviceBuf out;                    // device result
  PinnedBuf stage[kStageBufs];      // pinned D2H staging ring
  cudaEvent_t ready[kStageBufs] = {};
  cudaStream_t stream = nullptr;
};

// Staged tables of the drop-in, keyed by a content hash and verified against
// the full table bytes on every hit (a hash collision never serves another
// dataset's tables); least recently used entries beyond kSliceCacheMax are
// destroyed, so a sweep over many triples keeps bounded HBM.
constexpr size_t kSliceCacheMax = 16;
struct SliceEntry {
  std::string bytes;  // the table arrays, concatenated as hashed
  pm2l_tables* tables = nullptr;
  uint64_t last_use = 0;
};
struct SliceCache {
  std::mutex mu;
  std::unordered_multimap<uint64_t, SliceEntry> tables;  // (content hash ^ device) -> staged
  uint64_t clock = 0;
  std::unordered_map<int, SliceDevice> dev;
  std::unique_ptr<CopyPool> pool;
};
SliceCache g_slice;

// Device result -> pageable caller buffer: chunked D2H into a ring of pinned
// buffers on `s`, each chunk copied out by the host pool while the next
// chunks are in flight over PCIe.
bool host_page_locked(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int drain_to_host(SliceDevice& sd, const double* d_out, double* out, size_t bytes) {
  if (!g_slice.pool) {
    // three quarters of the host threads (caller included): the copy-out is
    // host-memory-bound; on the 16-core B200 host 12 threads drain 80 MB in
    // 2.26 ms median against 2.51 with 8 and 2.24 with 16 (A/B, 3 runs each)
    const unsigned hc = std::thread::hardware_concurrency();
    int workers = int(std::min(15u, hc > 3 ? hc * 3 / 4 - 1 : 0u));
    if (const char* e = std::getenv("PM2L_COPY_THREADS")) workers = std::max(0, std::atoi(e) - 1);  // tuning
    g_slice.pool.reset(new CopyPool(workers));
  }
  const size_t kStageChunk = stage_chunk();
  for (int i = 0; i < kStageBufs; ++i) {
    PM2L_CUDA(sd.stage[i].reserve(kStageChunk));
    if (!sd.ready[i]) PM2L_CUDA(cudaEventCreateWithFlags(&sd.ready[i], cudaEventDisableTiming));
  }
  // chunk schedule: tapered at both ends so the host copy starts sooner and
  // the last copy, which nothing overlaps, is short; PM2L_STAGE_TAPER (read
  // once, tuning): 0 uniform C, 1 (default) or 2 levels of taper
  static const int taper = [] {
    const char* e = std::getenv("PM2L_STAGE_TAPER");
    return e ? std::atoi(e) : 1;
  }();
  std::vector<size_t> lens;
  {
    const size_t C = kStageChunk;
    size_t rest = bytes;
    const bool tp = taper > 0 && bytes > 3 * C;
    // level 1: head C/4, C/2; tail C/2, C/4, C/4.  level 2: head C/8, C/4,
    // C/2; tail C/2, C/4, C/8, C/8
    std::vector<size_t> head, tail;
    if (tp && taper == 1) { head = {C / 4, C / 2}; tail = {C / 2, C / 4, C / 4}; }
    if (tp && taper >= 2) { head = {C / 8, C / 4, C / 2}; tail = {C / 2, C / 4, C / 8, C / 8}; }
    size_t tail_bytes = 0;
    for (size_t h : tail) tail_bytes += h;
    for (size_t h : head) { lens.push_back(h); rest -= h; }
    while (rest > tail_bytes) {
      const size_t l = std::min(C, rest - tail_bytes);
      lens.push_back(l);
      rest -= l;
    }
    for (size_t h : tail) lens.push_back(h);
  }
  std::vector<size_t> offs(lens.size());
  for (size_t c = 0, o = 0; c < lens.size(); ++c) { offs[c] = o; o += lens[c]; }
  const size_t n = lens.size();
  auto issue = [&](size_t c) -> int {
    const size_t off = offs[c], len = lens[c];
    const int b = int(c % kStageBufs);
    PM2L_CUDA(cudaMemcpyAsync(sd.stage[b].ptr, reinterpret_cast<const uint8_t*>(d_out) + off, len,
                              cudaMemcpyDeviceToHost, sd.stream));
    PM2L_CUDA(cudaEventRecord(sd.ready[b], sd.stream));
    return PM2L_OK;
  };
  for (size_t c = 0; c < std::min<size_t>(n, kStageBufs); ++c)
    if (int rc = issue(c)) return rc;
  static const bool trace = std::getenv("PM2L_E2E_TRACE") != nullptr;  // diagnostics
  double t_wait = 0, t_copy = 0;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t_start = now();
  for (size_t c = 0; c < n; ++c) {
    const int b = int(c % kStageBufs);
    const auto t0 = now();
    PM2L_CUDA(cudaEventSynchronize(sd.ready[b]));
    const auto t1 = now();
    const size_t off = offs[c], len = lens[c];
    g_slice.pool->copy(reinterpret_cast<uint8_t*>(out) + off, sd.stage[b].ptr, len);
    t_wait += std::chrono::duration<double, std::milli>(t1 - t0).count();
    t_copy += std::chrono::duration<double, std::milli>(now() - t1).count();
    if (c + kStageBufs < n)
      if (int rc = issue(c + kStageBufs)) return rc;
  }
  if (trace)
    std::fprintf(stderr, "pm2l drain: %zu chunks, wait %.3f ms, copy %.3f ms, total %.3f ms\n", n,
                 t_wait, t_copy,
                 std::chrono::duration<double, std::milli>(now() - t_start).count());
  return PM2L_OK;
}

// The slice's latencies into a HOST buffer: the grid kernel writes the
// per-device result buffer, then a page-locked `out` takes one D2H copy and
// a pageable one the staged drain.  Synchronous.  Caller holds g_slice.mu.
int predict_to_host_locked(pm2l_tables* t, int device, const uint64_t* batch_vals,
                           int64_t n_batch, const uint64_t* m_vals, int64_t n_m,
                           const uint64_t* n_vals, int64_t n_n, const uint64_t* k_vals,
                           int64_t n_k, int64_t b_lo, int64_t b_hi, double* out) {
  SliceDevice& sd = g_slice.dev[device];
  cudaStream_t& s = sd.stream;
  if (!s) PM2L_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  if (b_lo < 0 || b_hi < b_lo || b_hi > n_batch || n_m < 0 || n_n < 0 || n_k < 0)
    return fail(PM2L_ERR_INVALID, "batch slice out of range");
  const int64_t count = (b_hi - b_lo) * n_m * n_n * n_k;
  if (count == 0) return PM2L_OK;
  if (!out) return fail(PM2L_ERR_INVALID, "null out");
  PM2L_CUDA(sd.out.reserve(size_t(count) * sizeof(double)));
  double* d_out = static_cast<double*>(sd.out.ptr);
  if (int rc = pm2l_grid_predict(t, batch_vals, n_batch, m_vals, n_m, n_vals, n_n, k_vals, n_k,
                                 b_lo, b_hi, d_out, nullptr, nullptr, nullptr, s))
    return rc;
  // a page-locked caller buffer (cudaHostAlloc / cudaHostRegister, e.g. a
  // pinned torch tensor's numpy view) takes the result straight from the
  // copy engine; pageable buffers go through the staged drain
  if (host_page_locked(out)) {
    PM2L_CUDA(cudaMemcpyAsync(out, d_out, size_t(count) * sizeof(double), cudaMemcpyDeviceToHost, s));
  } else if (int rc = drain_to_host(sd, d_out, out, size_t(count) * sizeof(double))) {
    return rc;
  }
  PM2L_CUDA(cudaStreamSynchronize(s));
  return PM2L_OK;
}

}  // namespace

int pm2l_predict_grid_slice(
    const uint64_t* batch_vals, int64_t n_batch, const uint64_t* m_vals, int64_t n_m,
    const uint64_t* n_vals, int64_t n_n, const uint64_t* k_vals, int64_t n_k, int64_t b_lo,
    int64_t b_hi, const uint64_t* exact_keys, const int64_t* exact_curve, int64_t n_records,
    const double* log_m, const double* log_n, const double* log_k, const int64_t* cand_curve,
    const int64_t* sample_offsets, const double* sample_dims, const double* sample_thrs,
    int64_t n_curves, const double* ref_dim, const double* ref_dur, const double* ref_thr,
    const double* ref_waves, const uint64_t* tile_m, const uint64_t* tile_n,
    const uint64_t* split_k, const uint64_t* blocks_per_wave, const uint8_t* family_rowblock,
    double* out) {
  NvtxRange nvtx_("pm2l_predict_grid_slice");
  if (int rc = check_device()) return rc;
  if (n_records < 0 || n_curves < 0 || !sample_offsets)
    return fail(PM2L_ERR_INVALID, "bad table sizes");
  int device = 0;
  PM2L_CUDA(cudaGetDevice(&device));
  pm2l_tables_view v{};
  v.n_records = n_records;
  v.exact_keys = exact_keys;
  v.exact_curve = exact_curve;
  v.log_m = log_m; v.log_n = log_n; v.log_k = log_k;
  v.cand_curve = cand_curve;
  v.n_curves = n_curves;
  v.sample_offsets = sample_offsets;
  v.sample_dims = sample_dims; v.sample_thrs = sample_thrs;
  v.ref_dim = ref_dim; v.ref_dur = ref_dur; v.ref_thr = ref_thr; v.ref_waves = ref_waves;
  v.tile_m = tile_m; v.tile_n = tile_n; v.split_k = split_k;
  v.blocks_per_wave = blocks_per_wave; v.family_rowblock = family_rowblock;

  const int64_t S = sample_offsets[n_curves];
  uint64_t h = 0xcbf29ce484222325ull ^ uint64_t(device);
  const size_t R = size_t(n_records), C = size_t(n_curves);
  std::string key;
  key.reserve(16 + 48 * R + 8 * (C + 1) + 16 * size_t(S > 0 ? S : 0) + 65 * C);
  auto add = [&](const void* p, size_t n) {
    h = fnv(h, p, n);
    key.append(static_cast<const char*>(p), n);
  };
  add(&n_records, 8); add(&n_curves, 8);
  if (R) {
    add(exact_keys, 8 * R); add(exact_curve, 8 * R);
    add(log_m, 8 * R); add(log_n, 8 * R); add(log_k, 8 * R);
    add(cand_curve, 8 * R);
  }
  add(sample_offsets, 8 * (C + 1));
  if (S > 0) { add(sample_dims, 8 * S); add(sample_thrs, 8 * S); }
  if (C) {
    add(ref_dim, 8 * C); add(ref_dur, 8 * C); add(ref_thr, 8 * C);
    add(ref_waves, 8 * C); add(tile_m, 8 * C); add(tile_n, 8 * C);
    add(split_k, 8 * C); add(blocks_per_wave, 8 * C);
    add(family_rowblock, C);
  }

  std::lock_guard<std::mutex> lk(g_slice.mu);
  pm2l_tables* t = nullptr;
  auto range = g_slice.tables.equal_range(h);
  for (auto it = range.first; it != range.second; ++it)
    if (it->second.bytes == key) {
      t = it->second.tables;
      it->second.last_use = ++g_slice.clock;
      break;
    }
  if (!t) {
    if (int rc = pm2l_tables_create(&v, device, &t)) return rc;
    while (g_slice.tables.size() >= kSliceCacheMax) {
      auto lru = g_slice.tables.begin();
      for (auto it = g_slice.tables.begin(); it != g_slice.tables.end(); ++it)
        if (it->second.last_use < lru->second.last_use) lru = it;
      pm2l_tables_destroy(lru->second.tables);
      g_slice.tables.erase(lru);
    }
    SliceEntry e;
    e.bytes.swap(key);
    e.tables = t;
    e.last_use = ++g_slice.clock;
    g_slice.tables.emplace(h, std::move(e));
  }
  return predict_to_host_locked(t, device, batch_vals, n_batch, m_vals, n_m, n_vals, n_n, k_vals,
                                n_k, b_lo, b_hi, out);
}

int pm2l_grid_predict_host(pm2l_tables* t, const uint64_t* batch_vals, int64_t n_batch,
                           const uint64_t* m_vals, int64_t n_m, const uint64_t* n_vals,
                           int64_t n_n, const uint64_t* k_vals, int64_t n_k, int64_t b_lo,
                           int64_t b_hi, double* out) {
  NvtxRange nvtx_("pm2l_grid_predict_host");
  if (!t) return fail(PM2L_ERR_INVALID, "null tables");
  DeviceGuard guard(t->device);
  std::lock_guard<std::mutex> lk(g_slice.mu);
  return predict_to_host_locked(t, t->device, batch_vals, n_batch, m_vals, n_m, n_vals, n_n,
                                k_vals, n_k, b_lo, b_hi, out);
}

}  // extern "C"
