// Per-SM pipe throughput probes for the prefill softmax design (not product
// code). One CTA of W warps on one SM, each warp looping over independent
// instruction chains; clock64 around the loop.
//   ex2_f32     ex2.approx.ftz.f32             (MUFU)
//   ex2_f16x2   ex2.approx.f16x2                (MUFU, two results per lane)
//   cvt_f16x2   cvt.rn.f16x2.f32                (F2FP)
//   fma_f32x2   fma.rn.f32x2                    (FFMA2)
//   max3_f32    max.f32 d, a, b, c              (3-input FMNMX)
//   tmem_ld     tcgen05.ld.32x32b.x32 + wait    (bytes / clk / SM)
// and the accuracy of ex2.approx.f16x2 over the softmax's input range.
// Build: nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2410_00428_b200/csrc \
//        scripts/pipe_probe.cu -o build/pipe_probe
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "tc_sm100.cuh"

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)


constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(512, 1) pipe_kernel(float* out, unsigned long long* cycles, float seed) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (OP == 5) {
    if (warp == 0) lkv::tc::tmem_alloc<512>(&tslot);
    lkv::tc::fence_before_sync();
  }
  __syncthreads();
  lkv::tc::fence_after_sync();
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-6f - 0.5f;
  uint32_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const __half2 x = __floats2half2_rn(a[i], a[i] * 0.5f);
    h[i] = *reinterpret_cast<const uint32_t*>(&x);
  }
  unsigned long long c0 = clock64();
  __syncthreads();
  c0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if constexpr (OP == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    } else if constexpr (OP == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
    } else if constexpr (OP == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(__uint_as_float(h[i])), "f"(__uint_as_float(h[(i + 1) & 7])));
    } else if constexpr (OP == 3) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        unsigned long long x, y;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[2 * i]), "f"(a[2 * i + 1]));
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x));
        asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(y) : "l"(x));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a[2 * i]), "=f"(a[2 * i + 1]) : "l"(y));
      }
    } else if constexpr (OP == 4) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 3) & 7]));
    } else if constexpr (OP == 5) {
      if (warp < 16) {
        float v[32];
        const uint32_t ta = tslot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 32;
        lkv::tc::tmem_ld32(ta, v);
        lkv::tc::tmem_wait_ld();
        a[it & 7] += v[it & 31];
      }
    }
  }
  __syncthreads();
  const unsigned long long c1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(h[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
  if (OP == 5) {
    lkv::tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) lkv::tc::tmem_free<512>(tslot);
  }
}

__global__ void ex2_f16_accuracy(float* worst_rel, float lo, float hi, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = lo + (hi - lo) * i / (n - 1);
  const __half2 hx = __floats2half2_rn(x, x);
  uint32_t u = *reinterpret_cast<const uint32_t*>(&hx), r;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(u));
  const __half2 hr = *reinterpret_cast<const __half2*>(&r);
  const float got = __low2float(hr);
  const double want_exact_x = exp2(static_cast<double>(x));                 // vs the f32 input
  const double want_f16_x = exp2(static_cast<double>(__low2float(hx)));      // vs the rounded f16 input
  const float e1 = static_cast<float>(fabs(got - want_exact_x) / want_exact_x);
  const float e2 = static_cast<float>(fabs(got - want_f16_x) / want_f16_x);
  atomicMax(reinterpret_cast<int*>(&worst_rel[0]), __float_as_int(e1));
  atomicMax(reinterpret_cast<int*>(&worst_rel[1]), __float_as_int(e2));
}

template <int OP>
void run(const char* name, int warps, double per_iter_elems_per_warp) {
  float* out;
  unsigned long long* cyc;
  CK(cudaMalloc(&out, 512 * sizeof(float)));
  CK(cudaMalloc(&cyc, sizeof(unsigned long long)));
  pipe_kernel<OP><<<1, warps * 32>>>(out, cyc, 1.0f);
  CK(cudaDeviceSynchronize());
  pipe_kernel<OP><<<1, warps * 32>>>(out, cyc, 1.0f);
  CK(cudaDeviceSynchronize());
  unsigned long long c = 0;
  CK(cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost));
  const double elems = per_iter_elems_per_warp * 32.0 * warps * kIters;
  printf("{\"probe\": \"%s\", \"warps\": %d, \"cycles\": %llu, \"per_clk_per_sm\": %.2f}\n", name, warps, c,
         elems / static_cast<double>(c));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ex2_f32 (results)", w, 8);
    run<1>("ex2_f16x2 (results)", w, 16);
    run<2>("cvt_f16x2 (f32 inputs)", w, 16);
    run<3>("fma_f32x2 (f32 lanes)", w, 16);
    run<4>("max3_f32 (instr)", w, 8);
  }
  for (int w : {4, 8, 16}) run<5>("tmem_ld_32x32b_x32 (bytes)", w, 32 * 4.0 / 1.0);
  float* wr;
  CK(cudaMalloc(&wr, 2 * sizeof(float)));
  for (float lo : {-1.f, -4.f, -16.f}) {
    CK(cudaMemset(wr, 0, 2 * sizeof(float)));
    const int n = 1 << 20;
    ex2_f16_accuracy<<<(n + 255) / 256, 256>>>(wr, lo, 0.f, n);
    float h[2];
    CK(cudaMemcpy(h, wr, sizeof h, cudaMemcpyDeviceToHost));
    printf("{\"probe\": \"ex2.approx.f16x2 accuracy\", \"x_range\": [%g, 0], \"max_rel_err_vs_f32_x\": %.3e, "
           "\"max_rel_err_vs_f16_x\": %.3e}\n", lo, h[0], h[1]);
  }
  return 0;
}
