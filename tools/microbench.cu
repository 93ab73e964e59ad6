// microbench.cu -- B200 measurements behind the rooflines of DESIGN.md §6
// (SURVEY.md §8(d) "Microbenchmarks the harness must run first"):
//   * L2 capacity attributes, L2-resident and HBM read bandwidth
//   * dependent-load latency (L2 hit, HBM)
//   * __syncthreads, barrier.cluster and grid-barrier (atomic flag) latency
//   * 64-bit integer multiply-add and 64-bit logic throughput (the op and hash ALU work)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
// Prints one JSON object.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                 \
      return 1;                                                               \
    }                                                                         \
  } while (0)

__global__ void k_read(const uint4* __restrict__ p, size_t n, size_t reps, uint4* out) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const uint4 v = __ldcg(p + i);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  if (acc.x == 0x12345678) out[0] = acc;
}

__global__ void k_chase(const uint32_t* __restrict__ next, uint32_t start, int steps, unsigned long long* cyc,
                        uint32_t* sink) {
  uint32_t i = start;
  const unsigned long long t0 = clock64();
  for (int s = 0; s < steps; ++s) i = __ldcg(next + i);
  const unsigned long long t1 = clock64();
  cyc[0] = t1 - t0;
  sink[0] = i;
}

// 8 independent chains per thread: a = a * b + c (64-bit; the fused hash term) or
// a = (a ^ b) & c | d (64-bit logic; the op evaluation), iters rounds.
template <int KIND>
__global__ void k_alu64(int iters, uint64_t seed, uint64_t* out) {
  uint64_t a[8], b = seed * 0x9E3779B97F4A7C15ull + threadIdx.x, c = b ^ 0x5EEDull, d = ~b;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = b + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (KIND == 0) a[k] = a[k] * b + c;
      else a[k] = ((a[k] ^ b) & c) | (d + a[k]);
    }
  }
  uint64_t r = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) r ^= a[k];
  if (r == 42) out[0] = r;
}

__global__ void k_syncthreads(int iters, unsigned long long* cyc) {
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_cluster_sync(int iters, unsigned long long* cyc) {
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_grid_sync(int iters, unsigned long long* bar, unsigned long long* cyc) {
  unsigned long long target = 0;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1ull);
      while (ld_acq(bar) < target) {
      }
      __threadfence();
    }
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_cg_grid_sync(int iters, unsigned long long* cyc) {
  auto g = cooperative_groups::this_grid();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  int dev = 0, sms = 0, l2 = 0, persist = 0, clk = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  uint4* buf = nullptr;
  uint4* out = nullptr;
  const size_t big = 4ull << 30;  // 4 GiB
  CK(cudaMalloc(&buf, big));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(buf, 1, big));
  printf("{\"sm_count\": %d, \"l2_bytes\": %d, \"l2_persisting_max_bytes\": %d, \"sm_clock_khz_attr\": %d", sms, l2,
         persist, clk);
  // read bandwidth vs working set
  printf(", \"read_bw_gbs\": {");
  const size_t sets[] = {8ull << 20, 32ull << 20, 64ull << 20, 96ull << 20, 2ull << 30};
  for (int k = 0; k < 5; ++k) {
    const size_t bytes = sets[k];
    const size_t n = bytes / 16;
    const size_t reps = bytes >= (1ull << 30) ? 2 : std::max<size_t>(1, (2ull << 30) / bytes);
    k_read<<<sms * 4, 512>>>(buf, n, 1, out);  // warm
    CK(cudaEventRecord(e0));
    k_read<<<sms * 4, 512>>>(buf, n, reps, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("%s\"%zu_MiB\": %.1f", k ? ", " : "", bytes >> 20, (double)bytes * reps / (ms * 1e-3) / 1e9);
  }
  printf("}");
  // dependent-load latency (random permutation cycle)
  for (int which = 0; which < 2; ++which) {
    const size_t n = which == 0 ? (16ull << 20) / 4 : (1ull << 30) / 4;  // 16 MiB (L2) / 1 GiB (HBM)
    std::vector<uint32_t> perm(n);
    for (size_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
    uint64_t x = 88172645463325252ull;
    for (size_t i = n - 1; i > 0; --i) {  // Sattolo: one big cycle
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      const size_t j = x % i;
      std::swap(perm[i], perm[j]);
    }
    uint32_t* d_next = reinterpret_cast<uint32_t*>(buf);
    CK(cudaMemcpy(d_next, perm.data(), n * 4, cudaMemcpyHostToDevice));
    unsigned long long* cyc = reinterpret_cast<unsigned long long*>(out);
    k_chase<<<1, 1>>>(d_next, 0, 20000, cyc, reinterpret_cast<uint32_t*>(out) + 8);  // warm
    k_chase<<<1, 1>>>(d_next, 1, 20000, cyc, reinterpret_cast<uint32_t*>(out) + 8);
    unsigned long long c = 0;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf(", \"%s_load_latency_cycles\": %.1f", which == 0 ? "l2" : "hbm", c / 20000.0);
  }
  CK(cudaMemset(buf, 1, 1 << 20));
  unsigned long long* cyc = reinterpret_cast<unsigned long long*>(out);
  unsigned long long c = 0;
  const int it = 2000;
  k_syncthreads<<<1, 1024>>>(it, cyc);
  CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
  printf(", \"syncthreads_1024_cycles\": %.1f", c / (double)it);
  for (int cs : {2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * (sms / cs));
    cfg.blockDim = dim3(768);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_cluster_sync, it, cyc));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf(", \"cluster%d_sync_cycles\": %.1f", cs, c / (double)it);
  }
  for (int grid : {1, 16, 74, 148}) {
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(buf);
    CK(cudaMemset(bar, 0, 8));
    void* args[] = {(void*)&it, (void*)&bar, (void*)&cyc};
    CK(cudaLaunchCooperativeKernel((void*)k_grid_sync, grid, 1024, args, 0, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf(", \"grid%d_flag_barrier_cycles\": %.1f", grid, c / (double)it);
  }
  {
    int grid = sms;
    void* args[] = {(void*)&it, (void*)&cyc};
    CK(cudaLaunchCooperativeKernel((void*)k_cg_grid_sync, grid, 1024, args, 0, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf(", \"grid%d_cg_sync_cycles\": %.1f", grid, c / (double)it);
  }
  {  // 64-bit ALU throughput, whole GPU (ops per second, one op = one 64-bit multiply-add / logic step)
    uint64_t* out;
    CK(cudaMalloc(&out, 8));
    const int iters = 1 << 14, blocks = sms * 8, threads = 256;
    for (int kind = 0; kind < 2; ++kind) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&]() {
        if (kind == 0) k_alu64<0><<<blocks, threads>>>(iters, 3, out);
        else k_alu64<1><<<blocks, threads>>>(iters, 3, out);
      };
      launch();
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 8;
      printf(", \"%s_gops\": %.1f", kind == 0 ? "int64_madd" : "int64_logic", ops / (ms * 1e-3) / 1e9);
    }
    cudaFree(out);
  }
  printf("}\n");
  return 0;
}
