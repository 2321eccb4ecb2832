// spectral.cuh -- problem.spectral_norm (problem.py:47-68) for a dense device
// matrix: power iteration on M'M from v = cos(k + 1/2) / |.|, stop when
// |est - prev| <= tol max(est, 1), return 1.01 est.  Three fixed-order
// kernels per iteration (M v by warp per row, M' w by thread per column,
// then |w| and the normalisation in one CTA), so the result is run-to-run
// deterministic; the host drives the stop test.
#pragma once
#include <cuda_runtime.h>

namespace rapdb_spec {

__global__ void init_v(double* v, long long cols) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < cols; k += (long long)gridDim.x * blockDim.x)
    v[k] = cos((double)k + 0.5);
}

// y[r] = sum_c M[r ld + c] x[c]: warp per row, lane-strided chains + butterfly
__global__ void mv_rows(const double* __restrict__ M, long long rows, long long cols, long long ld,
                        const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = w0; r < rows; r += nw) {
    const double* row = M + r * ld;
    double s = 0.0;
    for (long long c = lane; c < cols; c += 32) s = fma(row[c], x[c], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = s;
  }
}

// y[c] = sum_r M[r ld + c] x[r]: thread per column, rows in order
__global__ void mv_cols(const double* __restrict__ M, long long rows, long long cols, long long ld,
                        const double* __restrict__ x, double* __restrict__ y) {
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long r = 0; r < rows; ++r) s = fma(M[r * ld + c], x[r], s);
    y[c] = s;
  }
}

// one CTA of 1024 threads: sq = |w|^2 (thread-strided chains, then a fixed
// tree), nrm = sqrt(sq) to out[0]; with normalize, v = w / nrm
__global__ void norm_normalize(const double* __restrict__ w, double* __restrict__ v, long long cols,
                               double* out, int normalize) {
  __shared__ double red[1024];
  double s = 0.0;
  for (long long k = threadIdx.x; k < cols; k += blockDim.x) s = fma(w[k], w[k], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + o];
    __syncthreads();
  }
  const double nrm = sqrt(red[0]);
  if (threadIdx.x == 0) out[0] = nrm;
  if (normalize && nrm > 0.0)
    for (long long k = threadIdx.x; k < cols; k += blockDim.x) v[k] = w[k] / nrm;
}

}  // namespace rapdb_spec
