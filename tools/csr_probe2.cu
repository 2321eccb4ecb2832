// csr_probe2.cu -- gather-SpMV variants at BASELINE C3 shapes with random
// (hashed) column indices, to pick the factored path's row / R^T kernels.
//   R x    : 6.5e6 rows x 10 nnz, gathers from x (1e6 doubles, 8 MB)
//   R^T w  : 1e6 rows x 65 nnz, gathers from W (6.5e6 doubles, 52 MB), and the
//            same split into 2 row phases (each phase gathers from 26 MB)
// Variants (all sum each row in stored order, so all give the same bits):
//   stage320   warp stages 32 rows' (val, col) coalesced in shared memory,
//              lanes fold their row with 4 gathers in flight (the r01 kernel)
//   thread     thread per row, all of a row's loads issued before its gathers
//   tmapipe    warp double-buffers the next 32-row group's (val, col) range
//              with TMA bulk copies while it folds the current one
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/csr_probe2 tools/csr_probe2.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t pol_ef() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_ef(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int ld_ef(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// rows of nnz entries, columns hashed into [c_lo, c_lo + c_span), sorted-ish not needed
__global__ void gen(long long rows, int nnz, long long c_lo, long long c_span, long long* ptr, int* col, double* val) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    ptr[r] = r * nnz;
    if (r == rows - 1) ptr[rows] = rows * nnz;
    for (int t = 0; t < nnz; ++t) {
      unsigned long long h = (unsigned long long)(r * nnz + t) * 0x9E3779B97F4A7C15ull;
      h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
      col[r * nnz + t] = (int)(c_lo + (long long)(h % (unsigned long long)c_span));
      val[r * nnz + t] = 1.0 / (1.0 + t);
    }
  }
}

template <int CAP>
__global__ void __launch_bounds__(256) k_stage(long long rows, const long long* ptr, const int* col,
                                              const double* val, const double* x, double* y) {
  __shared__ double sv[8][CAP];
  __shared__ int sc[8][CAP];
  const uint64_t ef = pol_ef();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long gw = blockIdx.x * 8LL + w, nw = gridDim.x * 8LL;
  for (long long r0 = gw * 32; r0 < rows; r0 += nw * 32) {
    const long long r = r0 + lane;
    const long long kb = ptr[r0];
    const long long ke = ptr[min(r0 + 32, rows)];
    long long k = r < rows ? ptr[r] : ke;
    const long long k1 = r < rows ? ptr[r + 1] : ke;
    double s = 0.0;
    for (long long base = kb; base < ke; base += CAP) {
      const long long lim = min(base + CAP, ke);
      for (long long e = base + lane; e < lim; e += 32) {
        sv[w][e - base] = ld_ef(val + e, ef);
        sc[w][e - base] = ld_ef(col + e, ef);
      }
      __syncwarp();
      const long long kend = min(k1, lim);
      for (; k + 4 <= kend; k += 4) {
        double xv[4], vv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) { vv[t] = sv[w][k + t - base]; xv[t] = __ldcg(x + sc[w][k + t - base]); }
#pragma unroll
        for (int t = 0; t < 4; ++t) s = __dadd_rn(s, __dmul_rn(vv[t], xv[t]));
      }
      for (; k < kend; ++k) s = __dadd_rn(s, __dmul_rn(sv[w][k - base], __ldcg(x + sc[w][k - base])));
      __syncwarp();
    }
    if (r < rows) y[r] = s;
  }
}

template <int B>
__global__ void __launch_bounds__(256) k_thread(long long rows, const long long* ptr, const int* col,
                                               const double* val, const double* x, double* y) {
  const uint64_t ef = pol_ef();
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    long long k = ptr[r];
    const long long k1 = ptr[r + 1];
    double s = 0.0;
    for (; k < k1; k += B) {
      int c[B]; double v[B], xv[B];
#pragma unroll
      for (int t = 0; t < B; ++t) if (k + t < k1) { c[t] = ld_ef(col + k + t, ef); v[t] = ld_ef(val + k + t, ef); }
#pragma unroll
      for (int t = 0; t < B; ++t) if (k + t < k1) xv[t] = __ldcg(x + c[t]);
#pragma unroll
      for (int t = 0; t < B; ++t) if (k + t < k1) s = __dadd_rn(s, __dmul_rn(v[t], xv[t]));
    }
    y[r] = s;
  }
}

// TMA double buffer per warp: group g+1's (val, col) range [a, b) (rounded out
// to multiples of 4 entries; arrays padded) lands in buffer (g+1)&1 while
// the lanes fold group g.  CAP entries per buffer; a group wider than CAP
// falls back to direct loads for the excess.
template <int CAP>
__global__ void __launch_bounds__(256) k_tmapipe(long long rows, const long long* ptr, const int* col,
                                                const double* val, const double* x, double* y) {
  extern __shared__ __align__(128) unsigned char dsm[];
  double (*sv)[2][CAP] = reinterpret_cast<double (*)[2][CAP]>(dsm);
  int (*sc)[2][CAP] = reinterpret_cast<int (*)[2][CAP]>(dsm + 8 * 2 * CAP * 8);
  uint64_t (*bar)[2] = reinterpret_cast<uint64_t (*)[2]>(dsm + 8 * 2 * CAP * 12);
  const uint64_t ef = pol_ef();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long gw = blockIdx.x * 8LL + w, nw = gridDim.x * 8LL;
  if (lane == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[w][b])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](long long r0, int b) {
    if (r0 >= rows) return;
    const long long kb = ptr[r0] & ~3LL;
    long long ke = (ptr[min(r0 + 32, rows)] + 3) & ~3LL;
    if (ke - kb > CAP) ke = kb + CAP;
    const unsigned nb = (unsigned)(ke - kb);
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[w][b])), "r"(nb * 12u) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   :: "r"(smem_u32(&sv[w][b][0])), "l"(val + kb), "r"(nb * 8u), "r"(smem_u32(&bar[w][b])), "l"(ef) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                   :: "r"(smem_u32(&sc[w][b][0])), "l"(col + kb), "r"(nb * 4u), "r"(smem_u32(&bar[w][b])), "l"(ef) : "memory");
    }
  };
  unsigned phase[2] = {0, 0};
  long long r0 = gw * 32;
  issue(r0, 0);
  int b = 0;
  for (; r0 < rows; r0 += nw * 32, b ^= 1) {
    issue(r0 + nw * 32, b ^ 1);
    // wait for buffer b
    {
      const uint32_t a = smem_u32(&bar[w][b]);
      unsigned ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(a), "r"(phase[b]) : "memory");
      }
      phase[b] ^= 1;
    }
    const long long r = r0 + lane;
    const long long base = ptr[r0] & ~3LL;
    long long k = r < rows ? ptr[r] : 0;
    const long long k1 = r < rows ? ptr[r + 1] : 0;
    double s = 0.0;
    const long long lim = base + CAP;
    for (; k + 4 <= k1 && k + 4 <= lim; k += 4) {
      double xv[4], vv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) { vv[t] = sv[w][b][k + t - base]; xv[t] = __ldcg(x + sc[w][b][k + t - base]); }
#pragma unroll
      for (int t = 0; t < 4; ++t) s = __dadd_rn(s, __dmul_rn(vv[t], xv[t]));
    }
    for (; k < k1; ++k) {
      const bool in = k < lim;
      const double v = in ? sv[w][b][k - base] : ld_ef(val + k, ef);
      const int c = in ? sc[w][b][k - base] : ld_ef(col + k, ef);
      s = __dadd_rn(s, __dmul_rn(v, __ldcg(x + c)));
    }
    if (r < rows) y[r] = s;
    __syncwarp();   // every lane done with buffer b before it is refilled
  }
}

static size_t smem_of(int cap) { return (size_t)8 * 2 * cap * 12 + 8 * 2 * 8; }

int main() {
  int nsm;
  CK(cudaFuncSetAttribute(k_tmapipe<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_of(512)));
  CK(cudaFuncSetAttribute(k_tmapipe<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_of(1024)));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  struct Shape { const char* name; long long rows, xlen; int nnz; long long c_lo, c_span; };
  Shape shapes[] = {{"R x (6.5e6 x 10, x 8 MB)", 6500000, 1000000, 10, 0, 1000000},
                    {"R^T (1e6 x 65, W 52 MB)", 1000000, 6500000, 65, 0, 6500000},
                    {"R^T phase (1e6 x 33, 26 MB)", 1000000, 6500000, 33, 0, 3250000},
                    {"R^T phase (1e6 x 16, 13 MB)", 1000000, 6500000, 16, 0, 1625000}};
  for (auto& sh : shapes) {
    long long* ptr; int* col; double *val, *x, *y;
    const long long nnz = sh.rows * sh.nnz;
    CK(cudaMalloc(&ptr, (sh.rows + 1) * 8));
    CK(cudaMalloc(&col, (nnz + 64) * 4));
    CK(cudaMalloc(&val, (nnz + 64) * 8));
    CK(cudaMalloc(&x, sh.xlen * 8));
    CK(cudaMalloc(&y, sh.rows * 8));
    CK(cudaMemset(x, 0, sh.xlen * 8));
    gen<<<nsm * 8, 256>>>(sh.rows, sh.nnz, sh.c_lo, sh.c_span, ptr, col, val);
    CK(cudaDeviceSynchronize());
    const double bytes = nnz * 12.0 + sh.rows * 16.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* label, auto launch) {
      for (int i = 0; i < 2; ++i) launch();
      CK(cudaGetLastError());
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
      printf("%-30s %-26s %8.4f ms  %7.1f GB/s\n", sh.name, label, ms, bytes / ms / 1e6);
      fflush(stdout);
    };
    for (int bpsm : {4, 6, 8}) {
      char lab[64];
      snprintf(lab, sizeof lab, "stage320 b/sm=%d", bpsm);
      timeit(lab, [&] { k_stage<320><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
      snprintf(lab, sizeof lab, "tmapipe512 b/sm=%d", bpsm);
      if (bpsm <= 2) timeit(lab, [&] { k_tmapipe<512><<<nsm * bpsm, 256, smem_of(512)>>>(sh.rows, ptr, col, val, x, y); });
    }
    for (int bpsm : {8, 16}) {
      char lab[64];
      snprintf(lab, sizeof lab, "thread B=8 b/sm=%d", bpsm);
      timeit(lab, [&] { k_thread<8><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
      snprintf(lab, sizeof lab, "thread B=16 b/sm=%d", bpsm);
      timeit(lab, [&] { k_thread<16><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    }
    {
      char lab[64];
      snprintf(lab, sizeof lab, "tmapipe512 b/sm=4 (64w)");
      timeit(lab, [&] { k_tmapipe<512><<<nsm * 4, 256, smem_of(512)>>>(sh.rows, ptr, col, val, x, y); });
      snprintf(lab, sizeof lab, "tmapipe1024 b/sm=2");
      timeit(lab, [&] { k_tmapipe<1024><<<nsm * 2, 256, smem_of(1024)>>>(sh.rows, ptr, col, val, x, y); });
    }
    CK(cudaGetLastError());
    cudaFree(ptr); cudaFree(col); cudaFree(val); cudaFree(x); cudaFree(y);
  }
  return 0;
}
