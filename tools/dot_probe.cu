// Multi-dot (c = V^T w) variants at the K_A pass-1 shape (n = 150^3, k = 28):
// warp-owned vectors with U row blocks in flight and MINB CTAs/SM forced by
// __launch_bounds__, vs the bw_probe single-accumulator stream.  GB/s = bytes
// of V + w read / event time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dot_probe tools/dot_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#include "../paper_2109_01232_b200/csrc/common.cuh"

template <int KV, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_dot(const float* __restrict__ w, long long n,
                                                   const float* __restrict__ V, long long ldv, int k,
                                                   float* out) {
  constexpr int RB = 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[KV];
#pragma unroll
  for (int q = 0; q < KV; ++q) acc[q] = 0.f;
  for (long long base = (long long)blockIdx.x * U * RB; base < n; base += (long long)gridDim.x * U * RB) {
    float4 wv[U], v[U][KV];
#pragma unroll
    for (int b = 0; b < U; ++b) {
      const long long r = base + b * RB + lane * 4;
      const bool in = r < n;
      wv[b] = in ? __ldg(reinterpret_cast<const float4*>(w + r)) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < KV; ++q) {
        const int i = warp + 8 * q;
        v[b][q] = (in && i < k) ? __ldcs(reinterpret_cast<const float4*>(V + (size_t)i * ldv + r))
                                : make_float4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int b = 0; b < U; ++b)
#pragma unroll
      for (int q = 0; q < KV; ++q) {
        acc[q] = fmaf(v[b][q].x, wv[b].x, acc[q]);
        acc[q] = fmaf(v[b][q].y, wv[b].y, acc[q]);
        acc[q] = fmaf(v[b][q].z, wv[b].z, acc[q]);
        acc[q] = fmaf(v[b][q].w, wv[b].w, acc[q]);
      }
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < KV; ++q) s += acc[q];
  if (s == 1234.5f) out[0] = s;
}

// vector-split: the CTA's 8 warps split the row block, each warp covers all k
// vectors for its 128-row sub-block with KT = k accumulators per lane
template <int KT, int MINB>
__global__ void __launch_bounds__(256, MINB) k_dot_rows(const float* __restrict__ w, long long n,
                                                        const float* __restrict__ V, long long ldv, int k,
                                                        float* out) {
  const int lane = threadIdx.x & 31;
  float acc[KT];
#pragma unroll
  for (int q = 0; q < KT; ++q) acc[q] = 0.f;
  const long long stride = (long long)gridDim.x * 256 * 4;
  for (long long r = ((long long)blockIdx.x * 256 + threadIdx.x) * 4; r < n; r += stride) {
    const float4 wv = __ldg(reinterpret_cast<const float4*>(w + r));
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      if (q < k) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(V + (size_t)q * ldv + r));
        acc[q] = fmaf(v.x, wv.x, fmaf(v.y, wv.y, fmaf(v.z, wv.z, fmaf(v.w, wv.w, acc[q]))));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < KT; ++q) s += acc[q];
  if (s == 1234.5f && lane == 0) out[0] = s;
}

// the probe kernel + the library's reduction tail: per-CTA partials of k + 2
// columns and a fixed-order last-CTA finalisation (warp per column)
__device__ unsigned g_counter = 0;
template <int KV, int U, int MINB, int FIN>
__global__ void __launch_bounds__(256, MINB) k_dot_fin(const float* __restrict__ w, long long n,
                                                       const float* __restrict__ V, long long ldv, int k,
                                                       float* part, float* out) {
  constexpr int RB = 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[KV];
#pragma unroll
  for (int q = 0; q < KV; ++q) acc[q] = 0.f;
  for (long long base = (long long)blockIdx.x * U * RB; base < n; base += (long long)gridDim.x * U * RB) {
    float4 wv[U], v[U][KV];
#pragma unroll
    for (int b = 0; b < U; ++b) {
      const long long r = base + b * RB + lane * 4;
      const bool in = r < n;
      wv[b] = in ? __ldg(reinterpret_cast<const float4*>(w + r)) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < KV; ++q) {
        const int i = warp + 8 * q;
        v[b][q] = (in && i < k) ? __ldcs(reinterpret_cast<const float4*>(V + (size_t)i * ldv + r))
                                : make_float4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int b = 0; b < U; ++b)
#pragma unroll
      for (int q = 0; q < KV; ++q) {
        acc[q] = fmaf(v[b][q].x, wv[b].x, acc[q]);
        acc[q] = fmaf(v[b][q].y, wv[b].y, acc[q]);
        acc[q] = fmaf(v[b][q].z, wv[b].z, acc[q]);
        acc[q] = fmaf(v[b][q].w, wv[b].w, acc[q]);
      }
  }
  const int stride = k + 2;
#pragma unroll
  for (int q = 0; q < KV; ++q) {
    float a = acc[q];
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0 && warp + 8 * q < k) part[(size_t)blockIdx.x * stride + warp + 8 * q] = a;
  }
  if (!FIN) return;
  if (FIN == 3) {   // cluster of 8: DSMEM reduction, one partial per cluster, no grid finalize
    __shared__ float cs[80];
    cg::cluster_group cl = cg::this_cluster();
    __syncthreads();
    for (int c = threadIdx.x; c < stride; c += blockDim.x) cs[c] = part[(size_t)blockIdx.x * stride + c];
    cl.sync();
    if (cl.block_rank() == 0) {
      for (int c = threadIdx.x; c < stride; c += blockDim.x) {
        float t = 0.f;
        for (int r = 0; r < 8; ++r) t += cl.map_shared_rank(cs, r)[c];
        out[(size_t)(blockIdx.x / 8) * stride + c] = t;
      }
    }
    cl.sync();
    return;
  }
  if (FIN == 2) {
    extern __shared__ float dummy[];
    (void)dummy;
    mpg::grid_reduce_cols<32>(part, 1184, part + 1184 * 80, reinterpret_cast<unsigned*>(part + 1184 * 80 + 64 * 80),
                              stride, [&](int c, float v) { out[c] = v; });
    return;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&g_counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) g_counter = 0;
  for (int c = warp; c < stride; c += 8) {
    float s = 0.f;
    for (int p = lane; p < (int)gridDim.x; p += 32) s += __ldcg(part + (size_t)p * stride + c);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = s;
  }
}

template <typename F>
float time_it(F f, int reps = 30) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <int KV, int U, int MINB>
void run(const float* w, long long n, const float* V, long long ldv, int k, float* out, int sms) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dot<KV, U, MINB>, 256, 0);
  cudaFuncAttributes at; cudaFuncGetAttributes(&at, k_dot<KV, U, MINB>);
  const int G = sms * occ;
  float t = time_it([&] { k_dot<KV, U, MINB><<<G, 256>>>(w, n, V, ldv, k, out); });
  printf("warp-owned KV=%d U=%d minb=%d: regs %d occ %d  %7.0f GB/s  %.1f us\n", KV, U, MINB, at.numRegs, occ,
         (double)(k + 1) * n * 4 / t / 1e6, t * 1e3);
}

template <int KT, int MINB>
void run_rows(const float* w, long long n, const float* V, long long ldv, int k, float* out, int sms) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dot_rows<KT, MINB>, 256, 0);
  cudaFuncAttributes at; cudaFuncGetAttributes(&at, k_dot_rows<KT, MINB>);
  const int G = sms * occ;
  float t = time_it([&] { k_dot_rows<KT, MINB><<<G, 256>>>(w, n, V, ldv, k, out); });
  printf("row-owned KT=%d minb=%d: regs %d occ %d  %7.0f GB/s  %.1f us\n", KT, MINB, at.numRegs, occ,
         (double)(k + 1) * n * 4 / t / 1e6, t * 1e3);
}

template <int KV, int U, int MINB, int FIN>
void run_fin(const float* w, long long n, const float* V, long long ldv, int k, float* part, float* out, int sms) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dot_fin<KV, U, MINB, FIN>, 256, 0);
  int G = sms * occ;
  float t;
  if (FIN == 3) {
    G = G / 8 * 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G); cfg.blockDim = dim3(256); cfg.stream = 0;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k_dot_fin<KV, U, MINB, FIN>, &cfg);
    if (ncl * 8 < G) G = ncl * 8;
    cfg.gridDim = dim3(G);
    t = time_it([&] { cudaLaunchKernelEx(&cfg, k_dot_fin<KV, U, MINB, FIN>, w, n, V, ldv, k, part, out); });
  } else {
    t = time_it([&] { k_dot_fin<KV, U, MINB, FIN><<<G, 256>>>(w, n, V, ldv, k, part, out); });
  }
  occ = G;
  printf("warp-owned+partials KV=%d U=%d minb=%d fin=%d: grid %d  %7.0f GB/s  %.1f us\n", KV, U, MINB, FIN, occ,
         (double)(k + 1) * n * 4 / t / 1e6, t * 1e3);
}

int main() {
  const long long n = 3375000, ldv = 3375040;
  const int K = 51, k = 28;
  float *V, *w, *out;
  cudaMalloc(&V, sizeof(float) * ldv * K);
  cudaMalloc(&w, sizeof(float) * ldv);
  cudaMalloc(&out, 64);
  cudaMemset(V, 0, sizeof(float) * ldv * K);
  cudaMemset(w, 0, sizeof(float) * ldv);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 1, 1>(w, n, V, ldv, k, out, sms);
  run<4, 2, 1>(w, n, V, ldv, k, out, sms);
  run<4, 4, 1>(w, n, V, ldv, k, out, sms);
  run<4, 1, 6>(w, n, V, ldv, k, out, sms);
  run<4, 2, 6>(w, n, V, ldv, k, out, sms);
  run<4, 1, 8>(w, n, V, ldv, k, out, sms);
  run<4, 2, 8>(w, n, V, ldv, k, out, sms);
  run<4, 2, 4>(w, n, V, ldv, k, out, sms);
  run<4, 4, 4>(w, n, V, ldv, k, out, sms);
  float* part; cudaMalloc(&part, sizeof(float) * (1184 * 80 + 64 * 80 + 128));
  cudaMemset(part, 0, sizeof(float) * (1184 * 80 + 64 * 80 + 128));
  float* outv; cudaMalloc(&outv, sizeof(float) * 80);
  run_fin<4, 2, 1, 0>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 2, 1, 1>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 1, 6, 0>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 1, 6, 1>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 2, 1, 2>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 1, 6, 2>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 2, 4, 0>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 2, 4, 3>(w, n, V, ldv, k, part, outv, sms);
  run_fin<4, 1, 6, 3>(w, n, V, ldv, k, part, outv, sms);
  run_rows<32, 1>(w, n, V, ldv, k, out, sms);
  run_rows<32, 2>(w, n, V, ldv, k, out, sms);
  run_rows<32, 3>(w, n, V, ldv, k, out, sms);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
