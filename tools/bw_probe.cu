// HBM read-stream probe for the basis sweeps (K_A/K_B/K_C access pattern):
// k basis rows of ldv floats, each thread reads 16 B of every row at its
// offset, U rows per batch.  Reports GB/s (bytes read / event time).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) k_multi(const float* __restrict__ V, long long ldv, long long n,
                                               int k, const float* __restrict__ c, float* out) {
  float acc = 0.f;
  const long long nv = n / 4;
  for (long long g = blockIdx.x * 256LL + threadIdx.x; g < nv; g += (long long)gridDim.x * 256) {
    float4 u = make_float4(0, 0, 0, 0);
    int i = 0;
    for (; i + U <= k; i += U) {
      float4 v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) v[q] = __ldcs(reinterpret_cast<const float4*>(V + (size_t)(i + q) * ldv) + g);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        u.x = fmaf(v[q].x, c[i + q], u.x); u.y = fmaf(v[q].y, c[i + q], u.y);
        u.z = fmaf(v[q].z, c[i + q], u.z); u.w = fmaf(v[q].w, c[i + q], u.w);
      }
    }
    for (; i < k; ++i) {
      float4 v = __ldcs(reinterpret_cast<const float4*>(V + (size_t)i * ldv) + g);
      u.x = fmaf(v.x, c[i], u.x); u.y = fmaf(v.y, c[i], u.y);
      u.z = fmaf(v.z, c[i], u.z); u.w = fmaf(v.w, c[i], u.w);
    }
    acc += u.x + u.y + u.z + u.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

// contiguous per-CTA slices (like cta_rows) instead of grid-stride
template <int U>
__global__ void __launch_bounds__(256) k_multi_slice(const float* __restrict__ V, long long ldv, long long n,
                                                     int k, const float* __restrict__ c, float* out) {
  float acc = 0.f;
  const long long nv = n / 4;
  const long long g0 = blockIdx.x * nv / gridDim.x, g1 = (blockIdx.x + 1) * nv / gridDim.x;
  for (long long g = g0 + threadIdx.x; g < g1; g += 256) {
    float4 u = make_float4(0, 0, 0, 0);
    int i = 0;
    for (; i + U <= k; i += U) {
      float4 v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) v[q] = __ldcs(reinterpret_cast<const float4*>(V + (size_t)(i + q) * ldv) + g);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        u.x = fmaf(v[q].x, c[i + q], u.x); u.y = fmaf(v[q].y, c[i + q], u.y);
        u.z = fmaf(v[q].z, c[i + q], u.z); u.w = fmaf(v[q].w, c[i + q], u.w);
      }
    }
    for (; i < k; ++i) {
      float4 v = __ldcs(reinterpret_cast<const float4*>(V + (size_t)i * ldv) + g);
      u.x = fmaf(v.x, c[i], u.x); u.y = fmaf(v.y, c[i], u.y);
      u.z = fmaf(v.z, c[i], u.z); u.w = fmaf(v.w, c[i], u.w);
    }
    acc += u.x + u.y + u.z + u.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, long long n4) {
  for (long long g = blockIdx.x * 256LL + threadIdx.x; g < n4; g += (long long)gridDim.x * 256) b[g] = a[g];
}

template <typename F>
float time_it(F f, int reps = 20) {
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

int main() {
  const long long n = 3375000, ldv = 3375040;
  const int K = 51;
  float *V, *c, *out;
  cudaMalloc(&V, sizeof(float) * ldv * K);
  cudaMalloc(&c, sizeof(float) * 64);
  cudaMalloc(&out, 64);
  cudaMemset(V, 0, sizeof(float) * ldv * K);
  cudaMemset(c, 0, 256);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int k : {8, 27, 50}) {
    const double bytes = (double)k * n * 4;
    for (int per : {4, 6, 8}) {
      const int G = sms * per;
      float t4 = time_it([&] { k_multi<4><<<G, 256>>>(V, ldv, n, k, c, out); });
      float t8 = time_it([&] { k_multi<8><<<G, 256>>>(V, ldv, n, k, c, out); });
      float s4 = time_it([&] { k_multi_slice<4><<<G, 256>>>(V, ldv, n, k, c, out); });
      float s8 = time_it([&] { k_multi_slice<8><<<G, 256>>>(V, ldv, n, k, c, out); });
      printf("k=%2d ctas/sm=%d  stride U4 %6.0f U8 %6.0f | slice U4 %6.0f U8 %6.0f GB/s\n", k, per,
             bytes / t4 / 1e6, bytes / t8 / 1e6, bytes / s4 / 1e6, bytes / s8 / 1e6);
    }
  }
  const long long n4 = ldv * 25 / 4;
  float tc = time_it([&] { k_copy<<<sms * 8, 256>>>((const float4*)V, (float4*)(V + ldv * 25), n4); });
  printf("copy %.0f GB/s (read+write)\n", 2.0 * n4 * 16 / tc / 1e6);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
