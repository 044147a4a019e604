// Store-bandwidth microbenchmark (diagnostics): n f64 (argv[1], default 10 M: 80 MB) written after a
// 256 MiB flush, by (1) STG.128 grid-stride, (2) STG.128 streaming (.cs),
// (3) TMA bulk stores (cp.async.bulk.global.shared::cta) from shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_bw store_bw.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void stg(double2* o, size_t n2, double v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x)
    o[i] = make_double2(v, v);
}
__global__ void stg_cs(double2* o, size_t n2, double v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x)
    __stcs(o + i, make_double2(v, v));
}
// each warp: fill a 4 KB smem chunk once, then bulk-store it repeatedly
__global__ void tma(double* o, size_t nchunks, double v) {
  extern __shared__ __align__(128) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* buf = sm + warp * 512;  // 4 KB per warp
  for (int j = lane; j < 512; j += 32) buf[j] = v;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const size_t wid = blockIdx.x * size_t(blockDim.x / 32) + warp, nw = size_t(gridDim.x) * (blockDim.x / 32);
  if (lane == 0) {
    for (size_t c = wid; c < nchunks; c += nw) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(o + c * 512),
                   "r"(uint32_t(__cvta_generic_to_shared(buf))) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main(int argc, char** argv) {
  // argv[1]: doubles to write (default 10 M = C2's 80 MB; 120 M = mode X's 960 MB)
  const size_t n = argc > 1 ? size_t(strtoull(argv[1], nullptr, 10)) : 10000000, bytes = n * 8;
  double *out, *flush;
  cudaMalloc(&out, bytes);
  cudaMalloc(&flush, size_t(256) << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaFuncSetAttribute(tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int variant = 0; variant < 6; ++variant) {
    for (int flushmode = 0; flushmode < 2; ++flushmode) {
      float best = 1e9, tot = 0;
      int cnt = 0;
      for (int it = 0; it < 12; ++it) {
        if (flushmode) cudaMemsetAsync(flush, it, size_t(256) << 20);
        cudaEventRecord(e0);
        if (variant == 0) stg<<<sms * 8, 256>>>((double2*)out, n / 2, 1.0);
        if (variant == 1) stg_cs<<<sms * 8, 256>>>((double2*)out, n / 2, 1.0);
        if (variant == 2) tma<<<sms * 2, 256, 32 * 1024>>>(out, bytes / 4096, 1.0);
        if (variant == 3) tma<<<sms * 4, 256, 32 * 1024>>>(out, bytes / 4096, 1.0);
        if (variant == 4) tma<<<sms * 6, 256, 32 * 1024>>>(out, bytes / 4096, 1.0);
        if (variant == 5) stg<<<sms * 2, 256>>>((double2*)out, n / 2, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2) { best = ms < best ? ms : best; tot += ms; ++cnt; }
      }
      const char* names[] = {"stg128 x8/SM", "stg128.cs x8/SM", "tma 4KB x2 CTA/SM", "tma 4KB x4 CTA/SM",
                             "tma 4KB x6 CTA/SM", "stg128 x2/SM"};
      printf("%-20s %s  mean %6.1f us  best %6.1f us  -> %5.0f GB/s\n", names[variant],
             flushmode ? "flushed" : "warm   ", 1e3 * tot / cnt, 1e3 * best, bytes / (tot / cnt) / 1e6);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
