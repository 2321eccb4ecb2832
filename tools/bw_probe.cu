// bw_probe.cu -- HBM streaming microbenchmark for the Q-sweep design on B200.
// Variants over one read-only buffer of `gb` GB (fp64):
//   ldg      : grid-stride double2 loads, 8-way unrolled, reduce to a checksum
//   bulk     : 1-D TMA bulk copies into an S-stage smem ring, one consumer warp
//              per stage summing it (static contiguous partition per CTA)
//   bulkdyn  : same, tiles handed out by a global atomic counter
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_ldg(const double2* __restrict__ a, long long n2, double* out) {
  double s0 = 0, s1 = 0;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long st = (long long)gridDim.x * blockDim.x;
  for (; i + 7 * st < n2; i += 8 * st) {
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(a + i + k * st);
#pragma unroll
    for (int k = 0; k < 8; ++k) { s0 += v[k].x; s1 += v[k].y; }
  }
  for (; i < n2; i += st) { double2 v = __ldg(a + i); s0 += v.x; s1 += v.y; }
  if (s0 + s1 == 12345.678) out[0] = s0;
}

template <bool DYN>
__global__ void __launch_bounds__(288, 1) k_bulk(const double* __restrict__ a, long long nbytes, int stage_bytes,
                                                  int nst, unsigned long long* ctr, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (long long)nst * stage_bytes);
  uint64_t* empty = full + nst;
  __shared__ long long s_tile[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long long ntot = nbytes / stage_bytes;
  const long long t0 = DYN ? 0 : (long long)blockIdx.x * ntot / gridDim.x;
  const long long t1 = DYN ? 0 : (long long)(blockIdx.x + 1) * ntot / gridDim.x;
  const int ncw = nst < 8 ? nst : 8;
  if (warp == 8) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int posted = 0;
      for (unsigned seq = 0;; ++seq) {
        long long tile;
        if (posted) tile = -1;
        else if (DYN) tile = (long long)atomicAdd(ctr, 1ULL);
        else tile = t0 + seq;
        const unsigned s = seq % nst, use = seq / nst;
        if (use > 0) {
          unsigned ok = 0;
          while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(su32(&empty[s])), "r"((use - 1) & 1) : "memory");
        }
        const bool done = posted || (DYN ? tile >= ntot : tile >= t1);
        s_tile[s] = done ? -1 : tile;
        if (done) {   // one end marker per consumer warp
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
          if (++posted == ncw) break;
          continue;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32(sm + (long long)s * stage_bytes)), "l"((const char*)a + tile * stage_bytes),
                     "r"(stage_bytes), "r"(su32(&full[s])), "l"(pol) : "memory");
      }
    }
  } else if (warp < ncw) {
    double acc = 0;
    for (unsigned seq = warp;; seq += ncw) {
      const unsigned s = seq % nst, use = seq / nst;
      unsigned ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(su32(&full[s])), "r"(use & 1) : "memory");
      const long long tile = *(volatile long long*)&s_tile[s];
      if (tile < 0) break;
      const double2* p = (const double2*)(sm + (long long)s * stage_bytes);
      for (int k = lane; k < stage_bytes / 16; k += 32) { double2 v = p[k]; acc += v.x + v.y; }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 12345.678) out[0] = acc;
  }
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 6.4;
  const long long nbytes = (long long)(gb * 1e9) / 65536 * 65536;
  double* a;
  double* out;
  unsigned long long* ctr;
  cudaMalloc(&a, nbytes);
  cudaMalloc(&out, 64);
  cudaMalloc(&ctr, 64);
  cudaMemset(a, 0, nbytes);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int bs : {288, 512, 1024}) {
    for (int blocks_per_sm : {1, 2}) {
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(e0);
        k_ldg<<<nsm * blocks_per_sm, bs>>>((const double2*)a, nbytes / 16, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("ldg      threads=%4d blocks/SM=%d   %8.1f GB/s\n", bs, blocks_per_sm, nbytes / ms / 1e6);
    }
  }
  int cfgs[][3] = {{4096, 48, 1}, {8192, 24, 1}, {8192, 16, 1}, {12288, 16, 1}, {16384, 12, 1}, {32768, 6, 1},
                   {8192, 12, 2}, {4096, 24, 2}};
  for (auto& c : cfgs) {
    const int sb = c[0], ns = c[1], bps = c[2];
    const int smem = sb * ns + 2 * ns * 8;
    auto k = k_bulk<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      k<<<nsm * bps, 288, smem>>>(a, nbytes, sb, ns, ctr, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaError_t err = cudaGetLastError();
    cudaEventElapsedTime(&ms, e0, e1);
    printf("bulk stage=%6d nst=%2d ctas/SM=%d  %8.1f GB/s %s\n", sb, ns, bps, nbytes / ms / 1e6,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  }
  return 0;
}
