// bar_probe.cu -- grid-barrier latency on a persistent grid (one 256-thread
// CTA per SM, like rapdb_solver_kernel): variants of the counter barrier.
//   V0: the solver's gsync (syncthreads, fence, atomicAdd, volatile spin with
//       nanosleep(16), fence, syncthreads)
//   V1: red.release.gpu + ld.acquire.gpu spin, no nanosleep
//   V2: V1 with nanosleep(16)
//   V3: atom.add.acq_rel + ld.acquire spin, no separate fences
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bar_probe tools/bar_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_acqrel(unsigned long long* p, unsigned long long v) {
  unsigned long long r;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(v) : "memory");
  return r;
}

__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

template <int V>
__global__ void __launch_bounds__(256, 1) bar_kernel(unsigned long long* bar, int iters, double* sink) {
  __shared__ unsigned long long gen;
  if (threadIdx.x == 0) gen = 0;
  __syncthreads();
  double acc = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    // a little per-phase work so the barrier is not back to back
    acc = acc * 1.0000001 + 1.0;
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      gen += gridDim.x;
      if (V == 0) {
        __threadfence();
        atomicAdd(bar, 1ULL);
        volatile unsigned long long* vb = bar;
        while (*vb < gen) __nanosleep(16);
        __threadfence();
      } else if (V == 1 || V == 2) {
        red_rel(bar, 1ULL);
        while (ld_acq(bar) < gen) { if (V == 2) __nanosleep(16); }
      } else if (V == 3) {
        unsigned long long r = atom_acqrel(bar, 1ULL) + 1;
        while (r < gen) r = ld_acq(bar);
      } else if (V == 4) {   // last arriver releases a flag on another line
        const unsigned long long r = atom_acqrel(bar, 1ULL) + 1;
        if (r == gen) st_rel(bar + 16, gen);
        else while (ld_acq(bar + 16) < gen) {}
      } else {               // two-level: groups of 16 CTAs, then the group leaders
        const int grp = blockIdx.x >> 4;
        const int ngrp = (gridDim.x + 15) >> 4;
        const unsigned long long gsize = (unsigned long long)min(16, (int)gridDim.x - grp * 16);
        const unsigned long long epoch = gen / gridDim.x;
        const unsigned long long r = atom_acqrel(bar + 32 + 16 * grp, 1ULL) + 1;
        if (r == epoch * gsize) {
          const unsigned long long t = atom_acqrel(bar + 16, 1ULL) + 1;
          if (t == epoch * ngrp) st_rel(bar + 24, epoch);
        }
        while (ld_acq(bar + 24) < epoch) {}
      }
    }
    __syncthreads();
  }
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* bar;
  double* sink;
  CK(cudaMalloc(&bar, 64 * 1024));
  CK(cudaMalloc(&sink, nsm * 256 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  auto run = [&](const char* name, auto kern) {
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemset(bar, 0, 64 * 1024));
      void* args[] = {&bar, (void*)&iters, &sink};
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel((const void*)kern, dim3(nsm), dim3(256), args, 0, 0));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("%-44s %7.3f us per barrier\n", name, ms * 1e3 / iters);
    }
  };
  run("V0 fence+atomicAdd+volatile spin(ns16)+fence", bar_kernel<0>);
  run("V1 red.release + ld.acquire spin", bar_kernel<1>);
  run("V2 red.release + ld.acquire spin(ns16)", bar_kernel<2>);
  run("V3 atom.acq_rel + ld.acquire spin", bar_kernel<3>);
  run("V4 atom.acq_rel, last arriver st.release flag", bar_kernel<4>);
  run("V5 two-level (16-CTA groups) + flag", bar_kernel<5>);
  return 0;
}
