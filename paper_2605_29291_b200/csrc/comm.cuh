// Native constraint-shard exchange over NCCL.
//
// The reference has no parallel code; its only requirement on a parallel
// build is a fixed reduction order.  A plain ncclAllReduce
// sums in an order that depends on the algorithm/protocol NCCL picks (ring,
// tree, NVLS in-switch reduction), so the cross-rank sums here are
// *rank-ordered*: NCCL only moves bytes (all-gather, send/recv) and a kernel
// of this library adds the R contributions as ((p_0 + p_1) + p_2) + ... --
// the same association the emulated cluster and the in-kernel peer exchange
// use, so all three sharded paths give the same bits on every rank.
//
//  * short buffers (R * count <= kGatherMax doubles): one ncclAllGather of
//    the partials into [R][count] scratch, then the ordered sum;
//  * long buffers: a deterministic reduce-scatter (grouped ncclSend/ncclRecv:
//    rank j receives chunk j of every rank), the ordered sum of its chunk,
//    and an in-place ncclAllGather of the reduced chunks -- the same
//    2 (R-1)/R * count bytes per rank as a ring all-reduce.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace rcomm {

constexpr long long kGatherMax = 1LL << 20;   // doubles (8 MB of [R][count] scratch)

// dst[j] = src[0][j] + src[1][j] + ... + src[R-1][j], added in rank order
// (-fmad=false; additions only, so the order is the whole story).
__global__ void ordered_sum_kernel(const double* __restrict__ src, int R, long long stride,
                                   long long count, double* __restrict__ dst) {
  const long long step = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += step) {
    double acc = src[j];
    for (int r = 1; r < R; ++r) acc = acc + src[(long long)r * stride + j];
    dst[j] = acc;
  }
}

struct Scratch {
  double* buf = nullptr;
  long long cap = 0;   // doubles
  ~Scratch() {
    if (buf) cudaFree(buf);
  }
  cudaError_t reserve(long long doubles) {
    if (doubles <= cap) return cudaSuccess;
    if (buf) {
      cudaError_t e = cudaFree(buf);
      buf = nullptr;
      cap = 0;
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaMalloc(&buf, (size_t)doubles * sizeof(double));
    if (e == cudaSuccess) cap = doubles;
    return e;
  }
};

inline int grid_for(long long count, int nsm) {
  long long g = (count + 255) / 256;
  const long long cap = 4LL * (nsm > 0 ? nsm : 148);
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// In-place rank-ordered all-reduce of buf[0..count) on `stream`.  Returns
// 0 or an NCCL/CUDA error code (negative: CUDA).
inline int ordered_allreduce(ncclComm_t comm, int rank, int R, double* buf, long long count,
                             Scratch& sc, cudaStream_t stream, int nsm, const char** what) {
  if (R <= 1 || count <= 0) return 0;
  if ((long long)R * count <= kGatherMax) {
    cudaError_t ce = sc.reserve((long long)R * count);
    if (ce != cudaSuccess) { *what = cudaGetErrorString(ce); return -1; }
    ncclResult_t nr = ncclAllGather(buf, sc.buf, (size_t)count, ncclDouble, comm, stream);
    if (nr != ncclSuccess) { *what = ncclGetErrorString(nr); return (int)nr; }
    ordered_sum_kernel<<<grid_for(count, nsm), 256, 0, stream>>>(sc.buf, R, count, count, buf);
    ce = cudaGetLastError();
    if (ce != cudaSuccess) { *what = cudaGetErrorString(ce); return -1; }
    return 0;
  }
  const long long chunk = (count + R - 1) / R;
  const long long padded = chunk * R;
  // [send: padded][recv: padded][gather: padded]
  cudaError_t ce = sc.reserve(3 * padded);
  if (ce != cudaSuccess) { *what = cudaGetErrorString(ce); return -1; }
  double* send = sc.buf;
  double* recv = sc.buf + padded;
  double* gath = sc.buf + 2 * padded;
  ce = cudaMemcpyAsync(send, buf, (size_t)count * sizeof(double), cudaMemcpyDeviceToDevice, stream);
  if (ce == cudaSuccess && padded > count)
    ce = cudaMemsetAsync(send + count, 0, (size_t)(padded - count) * sizeof(double), stream);
  if (ce != cudaSuccess) { *what = cudaGetErrorString(ce); return -1; }
  ncclResult_t nr = ncclGroupStart();
  for (int r = 0; r < R && nr == ncclSuccess; ++r) {
    nr = ncclSend(send + (long long)r * chunk, (size_t)chunk, ncclDouble, r, comm, stream);
    if (nr == ncclSuccess) nr = ncclRecv(recv + (long long)r * chunk, (size_t)chunk, ncclDouble, r, comm, stream);
  }
  const ncclResult_t ge = ncclGroupEnd();
  if (nr == ncclSuccess) nr = ge;
  if (nr != ncclSuccess) { *what = ncclGetErrorString(nr); return (int)nr; }
  double* mine = gath + (long long)rank * chunk;
  ordered_sum_kernel<<<grid_for(chunk, nsm), 256, 0, stream>>>(recv, R, chunk, chunk, mine);
  ce = cudaGetLastError();
  if (ce != cudaSuccess) { *what = cudaGetErrorString(ce); return -1; }
  nr = ncclAllGather(mine, gath, (size_t)chunk, ncclDouble, comm, stream);
  if (nr != ncclSuccess) { *what = ncclGetErrorString(nr); return (int)nr; }
  ce = cudaMemcpyAsync(buf, gath, (size_t)count * sizeof(double), cudaMemcpyDeviceToDevice, stream);
  if (ce != cudaSuccess) { *what = cudaGetErrorString(ce); return -1; }
  return 0;
}

}  // namespace rcomm
