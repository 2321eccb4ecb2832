// csr_probe.cu -- SpMV variants at BASELINE C3 shapes (fp64 values, int32
// indices, int64 row pointers), to pick the factored path's kernels:
//   R x      : 6.5e6 rows x 1e6 cols, 10 nnz/row (uniform columns)
//   R^T w    : 1e6 rows x 6.5e6 cols, ~65 nnz/row (the transposed gather)
// Each variant sums its row in stored order (thread-level sequential) or in
// a fixed lane tree; timing with CUDA events, bytes = 12 B/nnz + 8 B/row.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o csr_probe tools/csr_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void gen_const(long long rows, int nnz_row, long long ncols, long long* ptr, int* col, double* val) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    ptr[r] = r * nnz_row;
    if (r == rows - 1) ptr[rows] = rows * nnz_row;
    for (int k = 0; k < nnz_row; ++k) {
      const unsigned long long h = mix(r * 131 + k);
      col[r * nnz_row + k] = (int)(h % ncols);
      val[r * nnz_row + k] = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
    }
  }
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
__device__ __forceinline__ uint64_t pol_ef() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// V0: thread per row, sequential
__global__ void __launch_bounds__(256) spmv_thread(long long rows, const long long* ptr, const int* col, const double* val,
                                                   const double* x, double* y) {
  const uint64_t ef = pol_ef();
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    long long k = ptr[r];
    const long long k1 = ptr[r + 1];
    double s = 0.0;
    for (; k + 4 <= k1; k += 4) {
      int c[4]; double v[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) { c[t] = ld_ef(col + k + t, ef); v[t] = ld_ef(val + k + t, ef); }
#pragma unroll
      for (int t = 0; t < 4; ++t) s = __dadd_rn(s, __dmul_rn(v[t], __ldcg(x + c[t])));
    }
    for (; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(ld_ef(val + k, ef), __ldcg(x + ld_ef(col + k, ef))));
    y[r] = s;
  }
}

// V1: L lanes per row (L = 2..32), lane-strided partial sums + butterfly
template <int L>
__global__ void __launch_bounds__(256) spmv_lanes(long long rows, const long long* ptr, const int* col, const double* val,
                                                  const double* x, double* y) {
  const uint64_t ef = pol_ef();
  const int lane = threadIdx.x & 31, sub = lane % L;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long g = tid / L, gw0 = (tid / 32) * (32 / L);
  const long long ng = (long long)gridDim.x * blockDim.x / L;
  for (long long t0 = gw0; t0 < rows; t0 += ng) {   // warp-uniform trip count
    const long long r = t0 + (g - gw0);
    double s = 0.0;
    if (r < rows) {
      const long long k0 = ptr[r], k1 = ptr[r + 1];
      long long k = k0 + sub;
      for (; k + L < k1; k += 2 * L) {
        const int c0 = ld_ef(col + k, ef), c1 = ld_ef(col + k + L, ef);
        const double v0 = ld_ef(val + k, ef), v1 = ld_ef(val + k + L, ef);
        const double x0 = __ldcg(x + c0), x1 = __ldcg(x + c1);
        s = fma(v0, x0, s);
        s = fma(v1, x1, s);
      }
      if (k < k1) s = fma(ld_ef(val + k, ef), __ldcg(x + ld_ef(col + k, ef)), s);
    }
#pragma unroll
    for (int o = L / 2; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (r < rows && sub == 0) y[r] = s;
  }
}

// V2: L lanes per row, U rows per lane group in flight at once (for low
// occupancy: the persistent solver runs 8 warps per SM)
template <int L, int U>
__global__ void __launch_bounds__(256) spmv_lanes_u(long long rows, const long long* ptr, const int* col,
                                                    const double* val, const double* x, double* y) {
  const uint64_t ef = pol_ef();
  const int lane = threadIdx.x & 31, sub = lane % L;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long g = tid / L, gw0 = (tid / 32) * (32 / L);
  const long long ng = (long long)gridDim.x * blockDim.x / L;
  for (long long t0 = gw0 * U; t0 < rows; t0 += ng * U) {
    long long k[U], k1[U];
    double s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long r = t0 + (g - gw0) * U + u;
      s[u] = 0.0;
      k[u] = r < rows ? ptr[r] + sub : 0;
      k1[u] = r < rows ? ptr[r + 1] : 0;
    }
    bool more = true;
    while (__any_sync(0xffffffffu, more)) {
      more = false;
      int c[U];
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k[u] < k1[u]) { c[u] = ld_ef(col + k[u], ef); v[u] = ld_ef(val + k[u], ef); }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k[u] < k1[u]) {
          s[u] = fma(v[u], __ldcg(x + c[u]), s[u]);
          k[u] += L;
          more = more || k[u] < k1[u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int o = L / 2; o >= 1; o >>= 1) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
      const long long r = t0 + (g - gw0) * U + u;
      if (r < rows && sub == 0) y[r] = s[u];
    }
  }
}

__device__ __forceinline__ double ld_el(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t pol_el() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// V3: the solver's thread-per-row (8-batch + 4 + 1, FMA-free), x gathers
// either plain L2 (.cg) or with an evict_last policy
template <bool XEL>
__global__ void __launch_bounds__(256) spmv_solver(long long rows, const long long* ptr, const int* col,
                                                  const double* val, const double* x, double* y) {
  const uint64_t ef = pol_ef();
  const uint64_t el = pol_el();
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
    long long k = ptr[r];
    const long long k1 = ptr[r + 1];
    double s = 0.0;
    for (; k + 8 <= k1; k += 8) {
      int c[8]; double v[8], xv[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) { c[t] = ld_ef(col + k + t, ef); v[t] = ld_ef(val + k + t, ef); }
#pragma unroll
      for (int t = 0; t < 8; ++t) xv[t] = XEL ? ld_el(x + c[t], el) : __ldcg(x + c[t]);
#pragma unroll
      for (int t = 0; t < 8; ++t) s = __dadd_rn(s, __dmul_rn(v[t], xv[t]));
    }
    for (; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(ld_ef(val + k, ef), XEL ? ld_el(x + ld_ef(col + k, ef), el) : __ldcg(x + ld_ef(col + k, ef))));
    y[r] = s;
  }
}

// V4: warp-cooperative coalesced staging: a warp takes 32 consecutive rows,
// copies their contiguous (val, col) range into its shared buffer with
// coalesced loads, then each lane sums its own row in stored order (FMA-free)
// -- the same bits as thread-per-row.  CAP entries per warp per pass.
template <int CAP, bool XEL>
__global__ void __launch_bounds__(256) spmv_warpstage(long long rows, const long long* ptr, const int* col,
                                                     const double* val, const double* x, double* y) {
  __shared__ double sv[8][CAP];
  __shared__ int sc[8][CAP];
  const uint64_t ef = pol_ef();
  const uint64_t el = pol_el();
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
        for (int t = 0; t < 4; ++t) {
          const int c = sc[w][k + t - base];
          vv[t] = sv[w][k + t - base];
          xv[t] = XEL ? ld_el(x + c, el) : __ldcg(x + c);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) s = __dadd_rn(s, __dmul_rn(vv[t], xv[t]));
      }
      for (; k < kend; ++k) {
        const int c = sc[w][k - base];
        s = __dadd_rn(s, __dmul_rn(sv[w][k - base], XEL ? ld_el(x + c, el) : __ldcg(x + c)));
      }
      __syncwarp();
    }
    if (r < rows) y[r] = s;
  }
}

int main(int argc, char** argv) {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  struct Shape { const char* name; long long rows, cols; int nnz; };
  Shape shapes[] = {{"R x   (6.5e6 x 1e6, 10/row)", 6500000, 1000000, 10},
                    {"R^T w (1e6 x 6.5e6, 65/row)", 1000000, 6500000, 65}};
  for (auto& sh : shapes) {
    long long* ptr; int* col; double *val, *x, *y;
    const long long nnz = sh.rows * sh.nnz;
    CK(cudaMalloc(&ptr, (sh.rows + 1) * 8));
    CK(cudaMalloc(&col, nnz * 4));
    CK(cudaMalloc(&val, nnz * 8));
    CK(cudaMalloc(&x, sh.cols * 8));
    CK(cudaMalloc(&y, sh.rows * 8));
    CK(cudaMemset(x, 0, sh.cols * 8));
    gen_const<<<nsm * 8, 256>>>(sh.rows, sh.nnz, sh.cols, ptr, col, val);
    CK(cudaDeviceSynchronize());
    // sort columns within each row (CSR from scipy is sorted): not needed for timing
    const double bytes = nnz * 12.0 + sh.rows * 16.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* label, auto launch) {
      for (int i = 0; i < 2; ++i) launch();
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
      printf("%-30s %-22s %8.4f ms  %7.1f GB/s\n", sh.name, label, ms, bytes / ms / 1e6);
    };
    for (int bpsm : {8, 16, 32}) {
      char lab[64]; snprintf(lab, sizeof lab, "thread/row b/sm=%d", bpsm);
      timeit(lab, [&] { spmv_thread<<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    }
    timeit("2 lanes/row", [&] { spmv_lanes<2><<<nsm * 16, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("4 lanes/row", [&] { spmv_lanes<4><<<nsm * 16, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("8 lanes/row", [&] { spmv_lanes<8><<<nsm * 16, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("16 lanes/row", [&] { spmv_lanes<16><<<nsm * 16, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("32 lanes/row", [&] { spmv_lanes<32><<<nsm * 16, 256>>>(sh.rows, ptr, col, val, x, y); });
    // one 256-thread CTA per SM, like the persistent solver
    timeit("1cta: thread/row", [&] { spmv_thread<<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 2 lanes", [&] { spmv_lanes<2><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 8 lanes", [&] { spmv_lanes<8><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 2 lanes x4", [&] { spmv_lanes_u<2, 4><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 2 lanes x8", [&] { spmv_lanes_u<2, 8><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 4 lanes x4", [&] { spmv_lanes_u<4, 4><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 8 lanes x4", [&] { spmv_lanes_u<8, 4><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 8 lanes x8", [&] { spmv_lanes_u<8, 8><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    timeit("1cta: 16 lanes x4", [&] { spmv_lanes_u<16, 4><<<nsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    for (int bpsm : {4, 8}) {
      char lab[64];
      snprintf(lab, sizeof lab, "solver x.cg b/sm=%d", bpsm);
      timeit(lab, [&] { spmv_solver<false><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
      snprintf(lab, sizeof lab, "solver x.el b/sm=%d", bpsm);
      timeit(lab, [&] { spmv_solver<true><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
      snprintf(lab, sizeof lab, "warpstage320 b/sm=%d", bpsm);
      timeit(lab, [&] { spmv_warpstage<320, false><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
      snprintf(lab, sizeof lab, "warpstage320 x.el b/sm=%d", bpsm);
      timeit(lab, [&] { spmv_warpstage<320, true><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
      snprintf(lab, sizeof lab, "warpstage128 b/sm=%d", bpsm);
      timeit(lab, [&] { spmv_warpstage<128, false><<<nsm * bpsm, 256>>>(sh.rows, ptr, col, val, x, y); });
    }
    CK(cudaGetLastError());
    cudaFree(ptr); cudaFree(col); cudaFree(val); cudaFree(x); cudaFree(y);
  }
  return 0;
}
