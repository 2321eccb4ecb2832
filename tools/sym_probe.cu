// sym_probe.cu -- standalone prototype of the packed-symmetric Q sweep
// (paper_2605_29291_b200/csrc/symsweep.cuh): correctness against a dense
// matvec and timing of stream + reduce at BASELINE shapes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I. -o sym_probe tools/sym_probe.cu
// usage: sym_probe n nmat [reps] [nstages]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "paper_2605_29291_b200/csrc/symsweep.cuh"

using namespace rapdb::sym;

namespace rapdb {
namespace sym {
// ---- half-unit streaming: a unit's sub-rows travel as separate ring slots
// (sub-row 0: sub-tiles (0,0),(0,1); sub-row 1: the rest), so a slot is held
// only while one sub-row is computed.  Same arithmetic, same order, same Pt
// slots as consume_unit.

// sub-tiles and doubles offset (inside the unit) of half h
__device__ __forceinline__ void unit_half(bool diag, int rs, int cs, int h, int& first, int& count) {
  if (diag) {
    if (h == 0) { first = 0; count = rs == 2 ? 2 : 1; }
    else { first = 2; count = 1; }
  } else {
    first = h * cs;
    count = cs;
  }
}

struct HalfState {           // per-warp registers carried between the halves of a unit
  double c0, c1, o1;
};

// half h of unit (bi, bj) held in shared memory at `tile` (its first stored
// sub-tile); writes the row part(s) it completes and, at the last half, the
// column part / diagonal block
__device__ __forceinline__ void consume_half(const Geom& g, const double* __restrict__ tile,
                                             const double* __restrict__ xs, int bi, int bj, int h,
                                             double* __restrict__ Pa, uint64_t pol, HalfState& hs) {
  const int lane = threadIdx.x & 31;
  int rs, cs;
  unit_subtiles(g, bi, bj, rs, cs);
  const double* xr = xs + bi * kB;
  const double* xc = xs + bj * kB;
  const long long nbB = g.nbB;
  if (bi == bj) {
    double* out = Pa + ((long long)bi * nbB + bi) * kB;
    if (h == 0) {
      double o0 = col_dot(tile, xr);
      hs.o1 = 0.0;
      if (rs == 2) {
        const double* T01 = tile + kTD;
        const double xj = xc[kT + lane];
        double v[32];
        double c = 0.0;
#pragma unroll
        for (int r = 0; r < kT; ++r) {
          const double q = T01[r * kT + lane];
          v[r] = q * xj;
          c = fma(q, xr[r], c);
        }
        o0 = o0 + transpose_reduce(v);
        hs.o1 = c;
      }
      st_keep(out + lane, o0, pol);
      if (rs == 1) st_keep(out + kT + lane, 0.0, pol);
    } else {
      st_keep(out + kT + lane, hs.o1 + col_dot(tile, xr + kT), pol);
    }
    return;
  }
  if (h == 0) { hs.c0 = 0.0; hs.c1 = 0.0; }
  const int sr = h;
  double v[32];
#pragma unroll
  for (int r = 0; r < kT; ++r) v[r] = 0.0;
  for (int sc = 0; sc < cs; ++sc) {
    const double* T = tile + sc * kTD;
    const double xj = xc[sc * kT + lane];
    const double* xi = xr + sr * kT;
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int r = 0; r < kT; r += 2) {
      const double2 xx = *reinterpret_cast<const double2*>(xi + r);
      const double q0 = T[r * kT + lane], q1 = T[(r + 1) * kT + lane];
      v[r] = fma(q0, xj, v[r]);
      v[r + 1] = fma(q1, xj, v[r + 1]);
      c0 = fma(q0, xx.x, c0);
      c1 = fma(q1, xx.y, c1);
    }
    if (sc == 0) hs.c0 = hs.c0 + (c0 + c1); else hs.c1 = hs.c1 + (c0 + c1);
  }
  double* outR = Pa + ((long long)bi * nbB + bj) * kB;
  st_keep(outR + sr * kT + lane, transpose_reduce(v), pol);
  if (h == rs - 1) {
    double* outC = Pa + ((long long)bj * nbB + bi) * kB;
    st_keep(outC + lane, hs.c0, pol);
    if (cs == 2) st_keep(outC + kT + lane, hs.c1, pol);
  }
}

}  // namespace sym
}  // namespace rapdb

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint64_t* b, unsigned par) {
  unsigned ok;
  asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
               : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  return ok;
}

__device__ double hval(long long a, long long r, long long c) {
  if (r > c) { long long t = r; r = c; c = t; }
  unsigned long long z = (unsigned long long)(a * 1000003 + r * 7919 + c * 104729 + 12345);
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return (double)(z >> 11) * (1.0 / 9007199254740992.0) - 0.5 + (r == c ? 2.0 : 0.0);
}


// Experiment only (nocomp == 3): consume_unit that skips the R writes of odd
// block columns and the C writes of odd block rows -- the partial-write volume
// and transpose count a 2x2 "super-unit" scheme would have (results wrong).
__device__ __forceinline__ void consume_unit_halfw(const Geom& g, const double* __restrict__ tile,
                                                   const double* __restrict__ xs, int bi, int bj,
                                                   double* __restrict__ Pa, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  int rs, cs;
  unit_subtiles(g, bi, bj, rs, cs);
  const double* xr = xs + bi * kB;
  const double* xc = xs + bj * kB;
  const long long nbB = g.nbB;
  if (bi == bj) { consume_unit(g, tile, xs, bi, bj, Pa, pol); return; }
  double c[2] = {0.0, 0.0};
  double* outR = Pa + ((long long)bi * nbB + bj) * kB;
  for (int sr = 0; sr < rs; ++sr) {
    double v[32];
#pragma unroll
    for (int r = 0; r < kT; ++r) v[r] = 0.0;
    for (int sc = 0; sc < cs; ++sc) {
      const double* T = tile + (sr * cs + sc) * kTD;
      const double xj = xc[sc * kT + lane];
      const double* xi = xr + sr * kT;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int r = 0; r < kT; r += 2) {
        const double2 xx = *reinterpret_cast<const double2*>(xi + r);
        const double q0 = T[r * kT + lane], q1 = T[(r + 1) * kT + lane];
        v[r] = fma(q0, xj, v[r]);
        v[r + 1] = fma(q1, xj, v[r + 1]);
        c0 = fma(q0, xx.x, c0);
        c1 = fma(q1, xx.y, c1);
      }
      c[sc] = c[sc] + (c0 + c1);
    }
    if (!(bj & 1)) st_keep(outR + sr * kT + lane, transpose_reduce(v), pol);
    else if (v[0] == 12345.678) outR[0] = v[1];
  }
  double* outC = Pa + ((long long)bj * nbB + bi) * kB;
  if (!(bi & 1)) for (int sc = 0; sc < cs; ++sc) st_keep(outC + sc * kT + lane, c[sc], pol);
  else if (c[0] == 12345.678) outC[0] = c[1];
}

__global__ void gen_dense(double* D, int n, long long nmat) {
  const long long tot = nmat * n * (long long)n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    const long long a = i / ((long long)n * n), rc = i - a * (long long)n * n;
    D[i] = hval(a, rc / n, rc % n);
  }
}

__global__ void dense_mv(const double* D, int n, long long nmat, const double* x, double* u) {
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long row = gw; row < nmat * n; row += nw) {
    const double* d = D + row * n;
    double s = 0;
    for (int c = lane; c < n; c += 32) s = fma(d[c], x[c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (!lane) u[row] = s;
  }
}

__global__ void __launch_bounds__(288, 1) phase_a(Geom g, const Unit* __restrict__ units, const double* __restrict__ Qp,
                                                  int nmat, const double* __restrict__ x, double* __restrict__ Pt,
                                                  int ns, int slot_bytes, int xs_bytes, int pf, int nocomp) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* xs = reinterpret_cast<double*>(sm);
  unsigned char* ring = sm + xs_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (long long)ns * slot_bytes);
  uint64_t* empty = full + ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int j = threadIdx.x; j < g.nbB * kB; j += blockDim.x) xs[j] = j < g.n ? x[j] : 0.0;
  __syncthreads();
  const long long total = (long long)nmat * g.upm;
  const int G = gridDim.x, b = blockIdx.x;
  const long long mine = total > b ? (total - 1 - b) / G + 1 : 0;
  const int ncw = ns < 8 ? ns : 8;
  const long long mat_doubles = g.spm * kTD;
  if (warp == 8) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      long long a = b / g.upm;
      int u = (int)(b - a * g.upm);
      // L2 prefetch cursor pf units ahead of the ring
      long long pa = a;
      int pu = u;
      for (int t = 0; t < pf; ++t) {
        if (t < mine) {
          const Unit un = units[pu];
          int rs, cs;
          const unsigned by = (unsigned)unit_subtiles(g, un.bi, un.bj, rs, cs) * kTD * 8;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(Qp + pa * mat_doubles + (long long)un.off * kTD), "r"(by) : "memory");
        }
        pu += G;
        while (pu >= g.upm) { pu -= g.upm; ++pa; }
      }
      int s = 0;
      unsigned use = 0;
      for (long long k = 0; k < mine; ++k) {
        if (pf > 0 && k + pf < mine) {
          const Unit un = units[pu];
          int rs, cs;
          const unsigned by = (unsigned)unit_subtiles(g, un.bi, un.bj, rs, cs) * kTD * 8;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(Qp + pa * mat_doubles + (long long)un.off * kTD), "r"(by) : "memory");
          pu += G;
          while (pu >= g.upm) { pu -= g.upm; ++pa; }
        }
        if (use > 0) while (!try_wait(&empty[s], (use - 1) & 1)) {}
        const Unit un = units[u];
        int rs, cs;
        const unsigned bytes = (unsigned)unit_subtiles(g, un.bi, un.bj, rs, cs) * kTD * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32(ring + (long long)s * slot_bytes)), "l"(Qp + a * mat_doubles + (long long)un.off * kTD),
                     "r"(bytes), "r"(su32(&full[s])), "l"(pol) : "memory");
        u += G;
        while (u >= g.upm) { u -= g.upm; ++a; }
        if (++s == ns) { s = 0; ++use; }
      }
    }
  } else if (warp < ncw) {
    long long gi = b + (long long)warp * G;
    long long a = gi / g.upm;
    int u = (int)(gi - a * g.upm);
    int s = warp;
    unsigned use = 0;
    const long long pstride = (long long)g.nbB * g.nbB * kB;
    const uint64_t keep = evict_last_policy();
    for (long long k = warp; k < mine; k += ncw) {
      while (!try_wait(&full[s], use & 1)) {}
      const Unit un = units[u];
      // nocomp 1: no compute (pure stream); 2: compute, partials of every
      // matrix into matrix 0's slots (L2-resident: no DRAM write traffic)
      if (nocomp == 3) consume_unit_halfw(g, reinterpret_cast<const double*>(ring + (long long)s * slot_bytes), xs,
                                          un.bi, un.bj, Pt + a * pstride, keep);
      else if (nocomp != 1) consume_unit(g, reinterpret_cast<const double*>(ring + (long long)s * slot_bytes), xs, un.bi, un.bj,
                   Pt + (nocomp == 2 ? 0 : a) * pstride, keep);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      u += ncw * G;
      while (u >= g.upm) { u -= g.upm; ++a; }
      s += ncw;
      while (s >= ns) { s -= ns; ++use; }
    }
  }
}


__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Stream + reduction fused: unit partials go to a ring of W matrix slots
// (L2-resident), a reducer warp per CTA reduces matrix a once all its units
// are written (cnt[a]) and publishes red[a]; writers of matrix a >= W wait for
// red[a - W] (slot reuse).  Counters are cumulative over sweeps (epoch E).
__global__ void __launch_bounds__(288, 1) phase_fused(Geom g, const Unit* __restrict__ units,
                                                      const double* __restrict__ Qp, int nmat,
                                                      const double* __restrict__ x, double* __restrict__ Pt,
                                                      int ns, int slot_bytes, int xs_bytes, int W, int* cnt,
                                                      int* red, int E, double* __restrict__ U) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* xs = reinterpret_cast<double*>(sm);
  unsigned char* ring = sm + xs_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (long long)ns * slot_bytes);
  uint64_t* empty = full + ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int j = threadIdx.x; j < g.nbB * kB; j += blockDim.x) xs[j] = j < g.n ? x[j] : 0.0;
  __syncthreads();
  const long long total = (long long)nmat * g.upm;
  const int G = gridDim.x, b = blockIdx.x;
  const long long mine = total > b ? (total - 1 - b) / G + 1 : 0;
  const int ncw = ns < 7 ? ns : 7;
  const long long mat_doubles = g.spm * kTD;
  const long long pstride = (long long)g.nbB * g.nbB * kB;
  const int cnt_done = (E + 1) * g.upm, red_done = (E + 1) * g.nbB;
  if (warp == 8) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      long long a = b / g.upm;
      int u = (int)(b - a * g.upm);
      int s = 0;
      unsigned use = 0;
      for (long long k = 0; k < mine; ++k) {
        if (use > 0) while (!try_wait(&empty[s], (use - 1) & 1)) {}
        const Unit un = units[u];
        int rs, cs;
        const unsigned bytes = (unsigned)unit_subtiles(g, un.bi, un.bj, rs, cs) * kTD * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32(ring + (long long)s * slot_bytes)), "l"(Qp + a * mat_doubles + (long long)un.off * kTD),
                     "r"(bytes), "r"(su32(&full[s])), "l"(pol) : "memory");
        u += G;
        while (u >= g.upm) { u -= g.upm; ++a; }
        if (++s == ns) { s = 0; ++use; }
      }
    }
  } else if (warp < ncw) {
    long long gi = b + (long long)warp * G;
    long long a = gi / g.upm;
    int u = (int)(gi - a * g.upm);
    int s = warp;
    unsigned use = 0;
    const uint64_t keep = evict_last_policy();
    for (long long k = warp; k < mine; k += ncw) {
      while (!try_wait(&full[s], use & 1)) {}
      const Unit un = units[u];
      if (a >= W) while (ld_acquire(red + (a - W)) < red_done) __nanosleep(32);   // slot reuse
      consume_unit(g, reinterpret_cast<const double*>(ring + (long long)s * slot_bytes), xs, un.bi, un.bj,
                   Pt + (a % W) * pstride, keep);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        __threadfence();
        atomicAdd(cnt + (a * 8 + (b & 7)) * 32, 1);   // 8 sub-counters per matrix, one 128-B line each
      }
      u += ncw * G;
      while (u >= g.upm) { u -= g.upm; ++a; }
      s += ncw;
      while (s >= ns) { s -= ns; ++use; }
    }
  } else if (warp == 7) {
    // reducer: items t = a * nbB + B, round-robin over CTAs, in increasing t
    const int nbB = g.nbB;
    for (long long t = b; t < (long long)nmat * nbB; t += G) {
      const long long a = t / nbB;
      const int B = (int)(t - a * nbB);
      for (;;) {
        int c = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) c += ld_acquire(cnt + (a * 8 + q) * 32);
        if (c >= cnt_done) break;
        __nanosleep(64);
      }
      const double2* p = reinterpret_cast<const double2*>(Pt + ((a % W) * nbB + B) * (long long)nbB * kB) + lane;
      double sx = 0.0, sy = 0.0;
      int K = 0;
      for (; K + 8 <= nbB; K += 8) {
        double2 tt[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) tt[q] = __ldcg(p + (K + q) * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) { sx += tt[q].x; sy += tt[q].y; }
      }
      for (; K < nbB; ++K) { const double2 t2 = __ldcg(p + K * 32); sx += t2.x; sy += t2.y; }
      const int r = B * kB + 2 * lane;
      if (r < g.n) U[a * g.n + r] = sx;
      if (r + 1 < g.n) U[a * g.n + r + 1] = sy;
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicAdd(red + a, 1);
      }
    }
  }
}

// Half-unit ring: 16 KB slots, each unit's sub-rows in consecutive slots;
// slot tags make any distance between a warp's slots safe (a wait starts only
// once the producer has tagged the slot with the expected sequence number).
__global__ void __launch_bounds__(256, 1) phase_half(Geom g, const Unit* __restrict__ units,
                                                     const double* __restrict__ Qp, int nmat,
                                                     const double* __restrict__ x, double* __restrict__ Pt,
                                                     int ns, int slot_bytes, int xs_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned tag[64];
  double* xs = reinterpret_cast<double*>(sm);
  unsigned char* ring = sm + xs_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (long long)ns * slot_bytes);
  uint64_t* empty = full + ns;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
      tag[s] = 0xffffffffu;
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int j = threadIdx.x; j < g.nbB * kB; j += blockDim.x) xs[j] = j < g.n ? x[j] : 0.0;
  __syncthreads();
  const long long total = (long long)nmat * g.upm;
  const int G = gridDim.x, b = blockIdx.x;
  const long long mine = total > b ? (total - 1 - b) / G + 1 : 0;
  const int ncw = 7;
  const long long mat_doubles = g.spm * kTD;
  const long long pstride = (long long)g.nbB * g.nbB * kB;
  volatile unsigned* vtag = tag;
  if (warp == 7) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      long long a = b / g.upm;
      int u = (int)(b - a * g.upm);
      unsigned q = 0;
      int s = 0;
      unsigned use = 0;
      for (long long k = 0; k < mine; ++k) {
        const Unit un = units[u];
        int rs, cs;
        unit_subtiles(g, un.bi, un.bj, rs, cs);
        const bool diag = un.bi == un.bj;
        const double* base = Qp + a * mat_doubles + (long long)un.off * kTD;
        for (int h = 0; h < rs; ++h) {
          int first, count;
          unit_half(diag, rs, cs, h, first, count);
          if (use > 0) while (!try_wait(&empty[s], (use - 1) & 1)) {}
          vtag[s] = q;
          const unsigned bytes = (unsigned)count * kTD * 8;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(su32(ring + (long long)s * slot_bytes)), "l"(base + (long long)first * kTD),
                       "r"(bytes), "r"(su32(&full[s])), "l"(pol) : "memory");
          ++q;
          if (++s == ns) { s = 0; ++use; }
        }
        u += G;
        while (u >= g.upm) { u -= g.upm; ++a; }
      }
    }
  } else {
    // every consumer walks the CTA's unit sequence to track slot numbers
    long long a = b / g.upm;
    int u = (int)(b - a * g.upm);
    unsigned q = 0;
    const uint64_t keep = evict_last_policy();
    HalfState hs;
    for (long long k = 0; k < mine; ++k) {
      const Unit un = units[u];
      const int rs = (2 * un.bi + 1 < g.nb32) ? 2 : 1;
      if ((int)(k % ncw) == warp) {
        for (int h = 0; h < rs; ++h) {
          const unsigned qq = q + h;
          const int s = (int)(qq % ns);
          while (vtag[s] != qq) {}
          while (!try_wait(&full[s], (qq / ns) & 1)) {}
          consume_half(g, reinterpret_cast<const double*>(ring + (long long)s * slot_bytes), xs, un.bi, un.bj, h,
                       Pt + a * pstride, keep, hs);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
      }
      q += rs;
      u += G;
      while (u >= g.upm) { u -= g.upm; ++a; }
    }
  }
}

__global__ void phase_b(Geom g, int nmat, const double* __restrict__ Pt, double* __restrict__ U) {
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int nbB = g.nbB;
  for (long long it = gw; it < (long long)nmat * nbB; it += nw) {
    const long long a = it / nbB;
    const int B = (int)(it - a * nbB);
    const double2* p = reinterpret_cast<const double2*>(Pt + (a * nbB + B) * (long long)nbB * kB) + lane;
    double sx = 0.0, sy = 0.0;
    int K = 0;
    for (; K + 4 <= nbB; K += 4) {
      const double2 t0 = __ldcg(p + (K + 0) * 32), t1 = __ldcg(p + (K + 1) * 32);
      const double2 t2 = __ldcg(p + (K + 2) * 32), t3 = __ldcg(p + (K + 3) * 32);
      sx += t0.x; sy += t0.y; sx += t1.x; sy += t1.y; sx += t2.x; sy += t2.y; sx += t3.x; sy += t3.y;
    }
    for (; K < nbB; ++K) { const double2 t = __ldcg(p + K * 32); sx += t.x; sy += t.y; }
    const int r = B * kB + 2 * lane;
    if (r < g.n) U[a * g.n + r] = sx;
    if (r + 1 < g.n) U[a * g.n + r + 1] = sy;
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 2000;
  const int nmat = argc > 2 ? atoi(argv[2]) : 201;
  const int reps = argc > 3 ? atoi(argv[3]) : 20;
  int ns = argc > 4 ? atoi(argv[4]) : 0;
  const int pf = argc > 5 ? atoi(argv[5]) : 0;
  const int nocomp = argc > 6 ? atoi(argv[6]) : 0;
  const Geom g = make_geom(n);
  std::vector<Unit> hu(g.upm);
  fill_units(g, hu.data());
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  double *D, *Qp, *Pt, *x, *U, *Uref;
  Unit* units;
  const long long dense_b = (long long)nmat * n * n * 8, packed_b = (long long)nmat * g.spm * kTD * 8;
  const long long pt_b = (long long)nmat * g.nbB * g.nbB * kB * 8;
  CK(cudaMalloc(&D, dense_b));
  CK(cudaMalloc(&Qp, packed_b));
  CK(cudaMalloc(&Pt, pt_b));
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&U, (long long)nmat * n * 8));
  CK(cudaMalloc(&Uref, (long long)nmat * n * 8));
  CK(cudaMalloc(&units, g.upm * sizeof(Unit)));
  CK(cudaMemcpy(units, hu.data(), g.upm * sizeof(Unit), cudaMemcpyHostToDevice));
  std::vector<double> hx(n);
  for (int i = 0; i < n; ++i) hx[i] = std::sin(0.37 * i + 1.0);
  CK(cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice));
  gen_dense<<<nsm * 8, 256>>>(D, n, nmat);
  pack_kernel<<<dim3(g.upm, nmat), 256>>>(g, units, D, n, (long long)n * n, Qp);
  dense_mv<<<nsm * 8, 256>>>(D, n, nmat, x, Uref);
  CK(cudaDeviceSynchronize());
  const int xs_bytes = ((g.nbB * kB * 8) + 127) / 128 * 128;
  const int slot = 4 * kTD * 8;
  if (ns <= 0) ns = (int)((227 * 1024 - xs_bytes - 1024) / slot);
  const int smem = xs_bytes + ns * slot + 2 * ns * 8;
  CK(cudaFuncSetAttribute(phase_a, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  float msa = 0, msb = 0;
  const int W = argc > 7 ? atoi(argv[7]) : 0;
  if (W < 0) {   // half-unit ring (16 KB slots)
    const int hslot = 2 * kTD * 8;
    const int hns = -W;
    const int hsmem = xs_bytes + hns * hslot + 2 * hns * 8;
    CK(cudaFuncSetAttribute(phase_half, cudaFuncAttributeMaxDynamicSharedMemorySize, hsmem));
    for (int it = 0; it < reps + 2; ++it) {
      cudaEventRecord(e0);
      phase_half<<<nsm, 256, hsmem>>>(g, units, Qp, nmat, x, Pt, hns, hslot, xs_bytes);
      cudaEventRecord(e1);
      phase_b<<<nsm * 4, 256>>>(g, nmat, Pt, U);
      cudaEventRecord(e2);
      CK(cudaEventSynchronize(e2));
      float a_, b_;
      cudaEventElapsedTime(&a_, e0, e1);
      cudaEventElapsedTime(&b_, e1, e2);
      if (it >= 2) { msa += a_; msb += b_; }
    }
    CK(cudaGetLastError());
    msa /= reps; msb /= reps;
    std::vector<double> hU((long long)nmat * n), hR((long long)nmat * n);
    CK(cudaMemcpy(hU.data(), U, hU.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hR.data(), Uref, hR.size() * 8, cudaMemcpyDeviceToHost));
    double err = 0, mx = 0;
    for (size_t i = 0; i < hU.size(); ++i) { err = fmax(err, fabs(hU[i] - hR[i])); mx = fmax(mx, fabs(hR[i])); }
    printf("half ns=%d n=%d nmat=%d: phaseA %.4f ms (%.1f GB/s packed)  phaseB %.4f  total %.4f ms  max|err| %.3e (max|u| %.3e)\n",
           hns, n, nmat, msa, packed_b / msa / 1e6, msb, msa + msb, err, mx);
    return 0;
  }
  if (W > 0) {   // fused stream + reduction with a W-matrix partial ring
    int *cnt, *red;
    CK(cudaMalloc(&cnt, nmat * 8 * 32 * 4));
    CK(cudaMalloc(&red, nmat * 4));
    CK(cudaMemset(cnt, 0, nmat * 8 * 32 * 4));
    CK(cudaMemset(red, 0, nmat * 4));
    CK(cudaFuncSetAttribute(phase_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int Wr = W < nmat ? W : nmat;
    for (int it = 0; it < reps + 2; ++it) {
      cudaEventRecord(e0);
      phase_fused<<<nsm, 288, smem>>>(g, units, Qp, nmat, x, Pt, ns, slot, xs_bytes, Wr, cnt, red, it, U);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float a_;
      cudaEventElapsedTime(&a_, e0, e1);
      if (it >= 2) msa += a_;
    }
    CK(cudaGetLastError());
    msa /= reps;
    std::vector<double> hU((long long)nmat * n), hR((long long)nmat * n);
    CK(cudaMemcpy(hU.data(), U, hU.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hR.data(), Uref, hR.size() * 8, cudaMemcpyDeviceToHost));
    double err = 0, mx = 0;
    for (size_t i = 0; i < hU.size(); ++i) { err = fmax(err, fabs(hU[i] - hR[i])); mx = fmax(mx, fabs(hR[i])); }
    printf("fused W=%d n=%d nmat=%d ns=%d: %.4f ms (%.1f GB/s packed, %.1f dense-equiv)  max|err| %.3e (max|u| %.3e)\n",
           Wr, n, nmat, ns, msa, packed_b / msa / 1e6, dense_b / msa / 1e6, err, mx);
    return 0;
  }
  for (int it = 0; it < reps + 2; ++it) {
    cudaEventRecord(e0);
    phase_a<<<nsm, 288, smem>>>(g, units, Qp, nmat, x, Pt, ns, slot, xs_bytes, pf, nocomp);
    cudaEventRecord(e1);
    phase_b<<<nsm * 4, 256>>>(g, nmat, Pt, U);
    cudaEventRecord(e2);
    CK(cudaEventSynchronize(e2));
    float a_, b_;
    cudaEventElapsedTime(&a_, e0, e1);
    cudaEventElapsedTime(&b_, e1, e2);
    if (it >= 2) { msa += a_; msb += b_; }
  }
  CK(cudaGetLastError());
  msa /= reps; msb /= reps;
  std::vector<double> hU((long long)nmat * n), hR((long long)nmat * n);
  CK(cudaMemcpy(hU.data(), U, hU.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hR.data(), Uref, hR.size() * 8, cudaMemcpyDeviceToHost));
  double err = 0, mx = 0;
  for (size_t i = 0; i < hU.size(); ++i) { err = fmax(err, fabs(hU[i] - hR[i])); mx = fmax(mx, fabs(hR[i])); }
  // dense-row sweep for comparison: warp-per-row ldg matvec
  cudaEventRecord(e0);
  for (int it = 0; it < 5; ++it) dense_mv<<<nsm * 8, 256>>>(D, n, nmat, x, Uref);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float msd;
  cudaEventElapsedTime(&msd, e0, e1);
  msd /= 5;
  printf("pf=%d n=%d nmat=%d ns=%d smem=%d  packed %.3f GB (dense %.3f GB, Pt %.1f MB)\n", pf, n, nmat, ns, smem,
         packed_b / 1e9, dense_b / 1e9, pt_b / 1e6);
  printf("phaseA %.4f ms (%.1f GB/s packed)  phaseB %.4f ms  total %.4f ms  dense-equiv %.1f GB/s\n", msa,
         packed_b / msa / 1e6, msb, msa + msb, dense_b / (msa + msb) / 1e6);
  printf("dense ldg matvec %.4f ms (%.1f GB/s)   max|err| %.3e  (max|u| %.3e)\n", msd, dense_b / msd / 1e6, err, mx);
  return 0;
}
