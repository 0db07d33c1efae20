// grid_barrier.cu — latency probe for the persistent small-problem kernel:
// cooperative_groups grid.sync() against a flat counter barrier
// (red.release.gpu + ld.acquire.gpu spin), and a dependent L2 load chain.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o grid_barrier grid_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_cg(int iters, uint64_t* out) {
  cg::grid_group g = cg::this_grid();
  g.sync();
  const uint64_t t0 = gtimer();
  for (int i = 0; i < iters; ++i) g.sync();
  const uint64_t t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

// flat barrier: one arrival counter, generation-based target (no reset)
__device__ __forceinline__ void flat_sync(unsigned* ctr, unsigned& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

__global__ void k_flat(int iters, unsigned* ctr, uint64_t* out) {
  unsigned target = 0;
  flat_sync(ctr, target);
  const uint64_t t0 = gtimer();
  for (int i = 0; i < iters; ++i) flat_sync(ctr, target);
  const uint64_t t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

// barrier + one global write/read round trip per phase (the pattern of a phase
// that publishes partials and reads everyone's)
__global__ void k_flat_rt(int iters, unsigned* ctr, double* buf, uint64_t* out) {
  unsigned target = 0;
  flat_sync(ctr, target);
  const uint64_t t0 = gtimer();
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) buf[blockIdx.x * 32 + threadIdx.x] = acc + i;
    flat_sync(ctr, target);
    if (threadIdx.x < gridDim.x) acc += buf[threadIdx.x * 32 + (i & 31)];
  }
  const uint64_t t1 = gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.0) out[1] = 1;
}

__global__ void k_chain(const unsigned* nxt, int steps, uint64_t* out) {
  unsigned i = 0;
  const uint64_t t0 = gtimer();
  for (int s = 0; s < steps; ++s) i = __ldcg(&nxt[i]);
  const uint64_t t1 = gtimer();
  out[0] = t1 - t0;
  out[1] = i;
}

int main() {
  uint64_t* d_out;
  unsigned* ctr;
  double* buf;
  cudaMalloc(&d_out, 64);
  cudaMalloc(&ctr, 64);
  cudaMalloc(&buf, 160 * 32 * 8);
  const int iters = 2000;
  for (int grid : {64, 128, 148}) {
    for (int threads : {256, 512}) {
      uint64_t h[2];
      void* args[] = {(void*)&iters, (void*)&d_out};
      cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args, 0, 0);
      cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
      const double cgus = h[0] / 1e3 / iters;
      cudaMemset(ctr, 0, 64);
      void* args2[] = {(void*)&iters, (void*)&ctr, (void*)&d_out};
      cudaLaunchCooperativeKernel((void*)k_flat, grid, threads, args2, 0, 0);
      cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
      const double flus = h[0] / 1e3 / iters;
      cudaMemset(ctr, 0, 64);
      void* args3[] = {(void*)&iters, (void*)&ctr, (void*)&buf, (void*)&d_out};
      cudaLaunchCooperativeKernel((void*)k_flat_rt, grid, threads, args3, 0, 0);
      cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
      const double rtus = h[0] / 1e3 / iters;
      printf("grid %3d x %3d: cg grid.sync %.3f us, flat barrier %.3f us, flat + publish/read %.3f us  (%s)\n",
             grid, threads, cgus, flus, rtus, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // dependent L2 chain (1 MB of indices, stride 4 KB)
  const int N = 1 << 18;
  unsigned* hn = new unsigned[N];
  for (int i = 0; i < N; ++i) hn[i] = (unsigned)((i + 1021) % N);
  unsigned* dn;
  cudaMalloc(&dn, N * 4);
  cudaMemcpy(dn, hn, N * 4, cudaMemcpyHostToDevice);
  k_chain<<<1, 1>>>(dn, 2000, d_out);  // warm L2
  k_chain<<<1, 1>>>(dn, 2000, d_out);
  uint64_t h[2];
  cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
  printf("dependent L2 load: %.1f ns\n", h[0] / 2000.0);
  return 0;
}
