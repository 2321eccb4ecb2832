// gather_probe.cu -- the ceiling of random 8-byte gathers on one B200, the
// bound of the factored path's CSR passes (BASELINE C3: 65 M gathers per
// pass from an 8 MB x or a 52 MB W-cache, both L2-resident).
// Variants (G gathers, hashed indices computed in registers unless noted):
//   ldg8      one 8-byte ld.global.cg per gather, U independent loads in flight
//   ldg8idx   the same with the index read from a coalesced int stream
//   ldg4      4-byte gathers (is the limit per request or per byte?)
//   ldg16     16-byte gathers (double2)
//   pair      lanes 2k, 2k+1 hit the same 128-byte line (wavefront sharing)
//   tma16     one 16-byte cp.async.bulk per gather into shared memory
//   ldgsts8   one 8-byte cp.async (LDGSTS) per gather into shared memory
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long mix(unsigned long long h) {
  h *= 0x9E3779B97F4A7C15ull; h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
  return h;
}
__device__ __forceinline__ double ldcg8(const double* p) { return __ldcg(p); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int U>
__global__ void __launch_bounds__(256) k_ldg8(const double* __restrict__ x, long long N, long long per_thread, double* out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double s = 0.0;
  for (long long i = 0; i < per_thread; i += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcg8(x + mix((unsigned long long)(t * per_thread + i + u)) % (unsigned long long)N);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 1.2345) out[0] = s;
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg8idx(const double* __restrict__ x, const int* __restrict__ idx, long long G, double* out) {
  const long long nt = gridDim.x * (long long)blockDim.x;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < G; i += U * nt) {
    int c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = i + u * nt < G ? __ldcs(idx + i + u * nt) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldcg8(x + c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 1.2345) out[0] = s;
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg4(const float* __restrict__ x, long long N, long long per_thread, double* out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  float s = 0.f;
  for (long long i = 0; i < per_thread; i += U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(x + mix((unsigned long long)(t * per_thread + i + u)) % (unsigned long long)N);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 1.2345f) out[0] = s;
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg16(const double2* __restrict__ x, long long N, long long per_thread, double* out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double s = 0.0;
  for (long long i = 0; i < per_thread; i += U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(x + mix((unsigned long long)(t * per_thread + i + u)) % (unsigned long long)N);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
  }
  if (s == 1.2345) out[0] = s;
}

// lanes 2k and 2k+1 read neighbours in the same 128-byte line
template <int U>
__global__ void __launch_bounds__(256) k_pair(const double* __restrict__ x, long long N, long long per_thread, double* out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long tp = t >> 1;
  double s = 0.0;
  for (long long i = 0; i < per_thread; i += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long line = mix((unsigned long long)(tp * per_thread + i + u)) % (unsigned long long)(N / 16);
      v[u] = ldcg8(x + line * 16 + (t & 1) * 7);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
  }
  if (s == 1.2345) out[0] = s;
}

// 16-byte bulk copies: every thread issues ROUNDS copies per phase into its own slots
template <int ROUNDS>
__global__ void __launch_bounds__(256) k_tma16(const double* __restrict__ x, long long N, long long per_thread, double* out) {
  __shared__ __align__(16) double buf[256 * ROUNDS * 2];
  __shared__ __align__(8) uint64_t bar;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const uint32_t b = smem_u32(&bar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  double s = 0.0;
  unsigned phase = 0;
  for (long long i = 0; i < per_thread; i += ROUNDS) {
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(256 * ROUNDS * 16) : "memory");
    __syncthreads();
#pragma unroll
    for (int u = 0; u < ROUNDS; ++u) {
      const unsigned long long e = mix((unsigned long long)(t * per_thread + i + u)) % (unsigned long long)(N / 2);
      const uint32_t d = smem_u32(buf + (threadIdx.x * ROUNDS + u) * 2);
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                   :: "r"(d), "l"(x + e * 2), "r"(b) : "memory");
    }
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"(phase) : "memory");
    phase ^= 1;
#pragma unroll
    for (int u = 0; u < ROUNDS; ++u) s += buf[(threadIdx.x * ROUNDS + u) * 2];
    __syncthreads();
  }
  if (s == 1.2345) out[0] = s;
}

template <int ROUNDS>
__global__ void __launch_bounds__(256) k_ldgsts8(const double* __restrict__ x, long long N, long long per_thread, double* out) {
  __shared__ __align__(16) double buf[256 * ROUNDS];
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double s = 0.0;
  for (long long i = 0; i < per_thread; i += ROUNDS) {
#pragma unroll
    for (int u = 0; u < ROUNDS; ++u) {
      const unsigned long long e = mix((unsigned long long)(t * per_thread + i + u)) % (unsigned long long)N;
      const uint32_t d = smem_u32(buf + u * 256 + threadIdx.x);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(x + e) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int u = 0; u < ROUNDS; ++u) s += buf[u * 256 + threadIdx.x];
  }
  if (s == 1.2345) out[0] = s;
}

__global__ void k_fill_idx(int* idx, long long G, long long N) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < G; i += (long long)gridDim.x * blockDim.x)
    idx[i] = (int)(mix((unsigned long long)i) % (unsigned long long)N);
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  const int nsm = pr.multiProcessorCount;
  const long long G = 65000000;
  double *x, *out; int* idx;
  const long long Nmax = 6500000;
  CK(cudaMalloc(&x, Nmax * 8 + 256)); CK(cudaMemset(x, 0, Nmax * 8 + 256));
  CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&idx, G * 4));
  printf("{\"sm\": %d, \"gathers\": %lld, \"results\": [\n", nsm, G);
  bool first = true;
  auto rep = [&](const char* name, long long N, int cps, float ms, long long g) {
    printf("%s {\"variant\": \"%s\", \"vector_mb\": %.1f, \"ctas_per_sm\": %d, \"ms\": %.4f, \"ggather_s\": %.1f, \"gathers_per_clk_sm_at_1p7ghz\": %.3f}",
           first ? "" : ",\n", name, N * 8 / 1e6, cps, ms, g / ms / 1e6, g / (ms * 1e-3) / nsm / 1.7e9);
    first = false;
  };
  for (long long N : {1000000LL, 6500000LL}) {
    for (int cps : {2, 4, 8}) {
      const int grid = nsm * cps;
      const long long nt = grid * 256LL;
      const long long per = (G / nt) / 16 * 16;
      const long long g = per * nt;
      rep("ldg8_u8", N, cps, timeit([&] { k_ldg8<8><<<grid, 256>>>(x, N, per, out); }), g);
      rep("ldg8_u16", N, cps, timeit([&] { k_ldg8<16><<<grid, 256>>>(x, N, per, out); }), g);
      if (cps == 8) {
        rep("ldg4_u8", N, cps, timeit([&] { k_ldg4<8><<<grid, 256>>>((const float*)x, N * 2, per, out); }), g);
        rep("ldg16_u8", N, cps, timeit([&] { k_ldg16<8><<<grid, 256>>>((const double2*)x, N / 2, per, out); }), g);
        rep("pair_u8", N, cps, timeit([&] { k_pair<8><<<grid, 256>>>(x, N, per, out); }), g);
        k_fill_idx<<<nsm * 8, 256>>>(idx, G, N);
        rep("ldg8idx_u8", N, cps, timeit([&] { k_ldg8idx<8><<<grid, 256>>>(x, idx, G, out); }), G);
        rep("ldgsts8_r8", N, cps, timeit([&] { k_ldgsts8<8><<<grid, 256>>>(x, N, per, out); }), g);
      }
      if (cps <= 4) {
        rep("tma16_r4", N, cps, timeit([&] { k_tma16<4><<<grid, 256>>>(x, N, per / 4, out); }, 2), g / 4);
      }
    }
  }
  printf("\n]}\n");
  return 0;
}
