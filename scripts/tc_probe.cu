// Probe of the tcgen05 operand layouts used by the GQA tiles (not product
// code): four single-CTA MMAs checked against a CPU fp32 product.
//   T1  S^T[128x16]  = K[128 tok x 128 d] (K-major SW128, TMA 16-row boxes) . Q^T (K-major none)
//   T2  O^T[128x16]  = V^T (MN-major SW128, TMA) . P^T (MN-major none)
//   T3  S[128x128]   = Q (K-major SW128, TMA) . K^T (K-major SW128, TMA)
//   T4  O[128x128]   = P (K-major SW128, st.shared) . V (MN-major SW128, TMA)
//   T5  O[128x128]   = P (TMEM, tcgen05.st; TS form) . V (MN-major SW128, TMA)
//   T6  as T5 with P in fp16 and V in bf16 (mixed A/B formats of kind::f16)
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_2410_00428_b200/csrc
//        scripts/tc_probe.cu -o build/tc_probe
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_sm100.cuh"

using namespace lkv::tc;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

struct alignas(1024) Smem {
  uint8_t a[32768];
  uint8_t b[32768];
  uint64_t bar_tma, bar_mma;
  uint32_t tmem;
};

template <int TEST>
__global__ void __launch_bounds__(128, 1)
    probe_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const __nv_bfloat16* __restrict__ bsrc, float* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    bar_init(&s.bar_tma, 1);
    bar_init(&s.bar_mma, 1);
    bar_fence_init();
  }
  if (warp == 0) tmem_alloc<256>(&s.tmem);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = s.tmem;

  // ---- operand staging
  uint32_t tx = 0;
  if (tid == 0) {
    if (TEST == 1 || TEST == 2) {
      tx = 32768;
      bar_expect_tx(&s.bar_tma, tx);
      for (int h = 0; h < 2; ++h)
        for (int b = 0; b < 8; ++b) tma_load_2d(s.a + h * 16384 + b * 2048, &mapA, h * 64, b * 16, &s.bar_tma);
    } else if (TEST == 3) {
      tx = 65536;
      bar_expect_tx(&s.bar_tma, tx);
      for (int h = 0; h < 2; ++h) {
        tma_load_2d(s.a + h * 16384, &mapA, h * 64, 0, &s.bar_tma);
        tma_load_2d(s.b + h * 16384, &mapB, h * 64, 0, &s.bar_tma);
      }
    } else {  // T4, T5: V from A's data
      tx = 32768;
      bar_expect_tx(&s.bar_tma, tx);
      for (int h = 0; h < 2; ++h) tma_load_2d(s.b + h * 16384, &mapA, h * 64, 0, &s.bar_tma);
    }
  }
  // manual operands
  if (TEST == 1) {
    // Q [16 g][128 d] -> K-major, no swizzle: (g/8)*2048 + (d/8)*128 + (g%8)*16 + (d%8)*2
    for (int i = tid; i < 16 * 128; i += 128) {
      const int g = i / 128, d = i % 128;
      *reinterpret_cast<__nv_bfloat16*>(s.b + (g / 8) * 2048 + (d / 8) * 128 + (g % 8) * 16 + (d % 8) * 2) =
          bsrc[i];
    }
  } else if (TEST == 2) {
    // P^T [128 tok][16 g] -> MN-major, no swizzle: (t/8)*256 + (g/8)*128 + (t%8)*16 + (g%8)*2
    for (int i = tid; i < 128 * 16; i += 128) {
      const int t = i / 16, g = i % 16;
      *reinterpret_cast<__nv_bfloat16*>(s.b + (t / 8) * 256 + (g / 8) * 128 + (t % 8) * 16 + (g % 8) * 2) =
          bsrc[i];
    }
  } else if (TEST == 5 || TEST == 6) {
    // P [128 q][128 tok] -> TMEM columns [128, 192): lane = row, two bf16 per column
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + 128;
    for (int c = 0; c < 4; ++c) {
      uint32_t v[16];
      for (int i = 0; i < 16; ++i) v[i] = *reinterpret_cast<const uint32_t*>(bsrc + tid * 128 + c * 32 + 2 * i);
      tmem_st16(lane_addr + c * 16, v);
    }
    tmem_wait_st();
  } else if (TEST == 4) {
    // P [128 q][128 tok] -> K-major SW128, thread = row
    const int r = tid;
    for (int c = 0; c < 16; ++c) {
      uint4 v = *reinterpret_cast<const uint4*>(bsrc + r * 128 + c * 8);
      *reinterpret_cast<uint4*>(s.a + (c / 8) * 16384 + sw128_off(r, c % 8)) = v;
    }
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();

  if (tid == 0) {
    bar_wait(&s.bar_tma, 0);
    fence_after_sync();
    const uint32_t a0 = saddr(s.a), b0 = saddr(s.b);
    for (int kk = 0; kk < 8; ++kk) {
      uint64_t ad, bd;
      uint32_t id;
      if (TEST == 1) {
        ad = smem_desc(a0 + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, kLayoutSw128);
        bd = smem_desc(b0 + kk * 256, 128, 2048, kLayoutNone);
        id = idesc_bf16(128, 16, false, false);
      } else if (TEST == 2) {
        ad = smem_desc(a0 + kk * 2048, 16384, 1024, kLayoutSw128);
        bd = smem_desc(b0 + kk * 512, 256, 128, kLayoutNone);
        id = idesc_bf16(128, 16, true, true);
      } else if (TEST == 3) {
        ad = smem_desc(a0 + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, kLayoutSw128);
        bd = smem_desc(b0 + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, kLayoutSw128);
        id = idesc_bf16(128, 128, false, false);
      } else {
        ad = smem_desc(a0 + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024, kLayoutSw128);
        bd = smem_desc(b0 + kk * 2048, 16384, 1024, kLayoutSw128);
        id = idesc_bf16(128, 128, false, true);
      }
      if (TEST == 6) id = (id & ~(7u << 7));  // a_format = F16 (0), b_format stays BF16
      if (TEST == 5 || TEST == 6)
        mma_bf16_ts(tmem, tmem + 128 + kk * 8, bd, id, kk > 0);
      else
        mma_bf16(tmem, ad, bd, id, kk > 0);
    }
    mma_commit(&s.bar_mma);
  }
  __syncwarp();
  bar_wait(&s.bar_mma, 0);
  fence_after_sync();
  const int N = (TEST <= 2) ? 16 : 128;
  const uint32_t lane_addr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(lane_addr + c, v);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) out[tid * N + c + i] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

static float bf(const __nv_bfloat16& x) { return __bfloat162float(x); }

int main() {
  srand(7);
  auto rnd = [] { return __float2bfloat16((rand() / (float)RAND_MAX) * 2.f - 1.f); };
  std::vector<__nv_bfloat16> A(128 * 128), B(128 * 128), Bs(128 * 16);
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  for (auto& x : Bs) x = rnd();
  __nv_bfloat16 *dA, *dB, *dBs;
  float* dO;
  CK(cudaMalloc(&dA, A.size() * 2));
  CK(cudaMalloc(&dB, B.size() * 2));
  CK(cudaMalloc(&dBs, Bs.size() * 2));
  CK(cudaMalloc(&dO, 128 * 128 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dBs, Bs.data(), Bs.size() * 2, cudaMemcpyHostToDevice));
  CUtensorMap m16, m128A, m128B;
  if (!make_map_2d(&m16, dA, 128, 128, 256, 64, 16, true) || !make_map_2d(&m128A, dA, 128, 128, 256, 64, 128, true) ||
      !make_map_2d(&m128B, dB, 128, 128, 256, 64, 128, true)) {
    printf("tensor map encode failed\n");
    return 1;
  }
  const size_t smem = sizeof(Smem) + 1024;
  int fails = 0;
  std::vector<__half> Bh(128 * 128);
  for (size_t i = 0; i < B.size(); ++i) Bh[i] = __float2half(__bfloat162float(B[i]) * 0.999f);
  __half* dBh;
  CK(cudaMalloc(&dBh, Bh.size() * 2));
  CK(cudaMemcpy(dBh, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice));
  for (int test = 1; test <= 6; ++test) {
    CK(cudaMemset(dO, 0, 128 * 128 * 4));
    switch (test) {
      case 1:
        CK(cudaFuncSetAttribute(probe_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        probe_kernel<1><<<1, 128, smem>>>(m16, m16, dBs, dO);
        break;
      case 2:
        CK(cudaFuncSetAttribute(probe_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        probe_kernel<2><<<1, 128, smem>>>(m16, m16, dBs, dO);
        break;
      case 3:
        CK(cudaFuncSetAttribute(probe_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        probe_kernel<3><<<1, 128, smem>>>(m128A, m128B, dBs, dO);
        break;
      case 4:
        CK(cudaFuncSetAttribute(probe_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        probe_kernel<4><<<1, 128, smem>>>(m128A, m128B, dB, dO);
        break;
      case 5:
        CK(cudaFuncSetAttribute(probe_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        probe_kernel<5><<<1, 128, smem>>>(m128A, m128B, dB, dO);
        break;
      default:
        CK(cudaFuncSetAttribute(probe_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        probe_kernel<6><<<1, 128, smem>>>(m128A, m128B, reinterpret_cast<const __nv_bfloat16*>(dBh), dO);
        break;
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    const int N = test <= 2 ? 16 : 128;
    std::vector<float> O(128 * N);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < N; ++j) {
        double ref = 0;
        for (int k = 0; k < 128; ++k) {
          if (test == 1) ref += bf(A[i * 128 + k]) * bf(Bs[j * 128 + k]);          // K[tok i] . Q[g j]
          else if (test == 2) ref += bf(A[k * 128 + i]) * bf(Bs[k * 16 + j]);     // V[tok k][d i] * P^T[k][g j]
          else if (test == 3) ref += bf(A[i * 128 + k]) * bf(B[j * 128 + k]);     // Q[i] . K[j]
          else if (test == 6) ref += __half2float(Bh[i * 128 + k]) * bf(A[k * 128 + j]);  // fp16 P * bf16 V
          else ref += bf(B[i * 128 + k]) * bf(A[k * 128 + j]);                    // P[i][k] * V[k][j] (T4, T5)
        }
        maxerr = fmax(maxerr, fabs(ref - O[i * N + j]));
        maxref = fmax(maxref, fabs(ref));
      }
    const bool ok = maxerr < 1e-3 * fmax(1.0, maxref);
    fails += !ok;
    printf("T%d %s max_abs_err=%.3g max_ref=%.3g  O[0][0..3]=%.4f %.4f %.4f %.4f\n", test, ok ? "OK" : "FAIL",
           maxerr, maxref, O[0], O[1], O[2], O[3]);
  }
  printf("%s\n", fails ? "PROBE FAILED" : "PROBE OK");
  return fails ? 1 : 0;
}
