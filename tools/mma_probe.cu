// Probe: tcgen05.mma issue throughput per instruction shape, operands resident in smem (no TMA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_14883_b200/csrc
//        tools/mma_probe.cu -o /tmp/mma_probe
// Prints cycles per MMA for cta_group::1 M128 N{64,128,256} and cta_group::2 M256 N{128,256},
// with both operands K-major SW128, and with the B operand MN-major.
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100_ptx.cuh"

using namespace tp::ptx;

__device__ __forceinline__ void umma_cg1(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_cg1(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

template <int CG, int M, int N, bool B_MN>
__global__ void probe(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;            // 128 rows x 64 K (16 KB)
  uint8_t* sB = base + 16384;    // up to 256 rows x 64 K (32 KB)
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 16384 + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      tmem_alloc_cg2(slot, 512);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const bool leader = CG == 1 || cluster_rank() == 0;
  if (warp == 0 && threadIdx.x == 0 && leader) {
    constexpr uint32_t idesc = idesc_bf16_f32(M, N, false, B_MN);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = sdesc_sw128(a0 + k * 32, 16, 1024);
        const uint64_t bd = B_MN ? sdesc_sw128(b0 + k * 2048, 8192, 1024) : sdesc_sw128(b0 + k * 32, 16, 1024);
        if (CG == 1) umma_cg1(tmem, ad, bd, idesc, 1);
        else umma_bf16_cg2(tmem, ad, bd, idesc, 1);
      }
    }
    if (CG == 1) commit_cg1(bar); else umma_commit_cg2_mc(bar, 0x3);
    mbar_wait(bar, 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (CG == 2 && threadIdx.x == 0 && !leader) {
    mbar_wait(bar, 0);
  }
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else tmem_dealloc_cg2(tmem, 512);
  }
}

template <int CG, int M, int N, bool B_MN>
void run(const char* name, int grid) {
  unsigned long long* d;
  cudaMalloc(&d, 512 * 8);
  cudaMemset(d, 0, 512 * 8);
  const int smem = 16384 + 32768 + 1024 + 64;
  auto k = probe<CG, M, N, B_MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2000;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, d, reps);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, d, reps);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[512];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double mmas = 4.0 * reps;
  const double flops = 2.0 * M * N * 16 * mmas * (grid / CG);
  printf("%-28s grid %3d: %7.1f cycles/MMA  %8.1f TFLOP/s  (%s)\n", name, grid, mx / mmas,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<1, 128, 64, false>("cg1 M128 N64  K-major", 148);
  run<1, 128, 128, false>("cg1 M128 N128 K-major", 148);
  run<1, 128, 256, false>("cg1 M128 N256 K-major", 148);
  run<1, 128, 256, true>("cg1 M128 N256 B MN-major", 148);
  run<2, 256, 128, false>("cg2 M256 N128 K-major", 148);
  run<2, 256, 256, false>("cg2 M256 N256 K-major", 148);
  run<2, 256, 256, true>("cg2 M256 N256 B MN-major", 148);
  run<2, 256, 64, false>("cg2 M256 N64 K-major", 148);
  return 0;
}
