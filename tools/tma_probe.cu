// Probe: how fast can TMA fill one SM's shared memory, alone and under tcgen05.mma operand reads?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_14883_b200/csrc
//        tools/tma_probe.cu -o tools/tma_probe.bin -lcuda
// A persistent ring of STAGES stages, each stage = NBOX boxes of 64 bf16 (128 B, SW128) x ROWS rows
// from an L2-resident 4096 x 8192 bf16 matrix. Consumer modes: 0 = release immediately (raw fill
// rate), 1 = four cta_group::1 M128 N256 MMAs per stage reading A (first 16 KB) and B (next 32 KB).
// Prints per-SM bytes per SM clock and chip-wide TB/s for several grid sizes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100_ptx.cuh"

using namespace tp::ptx;

__device__ __forceinline__ void tma_load_cta(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
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

constexpr int kRows = 4096, kCols = 8192, kBigRows = 18944;

template <int STAGES, int NBOX, int ROWS, int MODE>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap map, int iters,
                                                unsigned long long* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int kBox = ROWS * 128;
  constexpr int kStage = NBOX * kBox;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint32_t* slot = reinterpret_cast<uint32_t*>(empty + STAGES);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  if (MODE == 1 && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int row_blocks = kRows / ROWS / NBOX;
  const int r0 = (blockIdx.x % row_blocks) * ROWS * NBOX;
  const int kblocks = kCols / 64;
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it)
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], kStage);
        for (int b = 0; b < NBOX; ++b)
          tma_load_cta(&map, &full[stage], sm + stage * kStage + b * kBox, kb * 64, r0 + b * ROWS);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
  } else if (threadIdx.x == 32) {
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t tmem = MODE == 1 ? *slot : 0;
    constexpr uint32_t idesc = idesc_bf16_f32(128, 256, false, false);
    for (int it = 0; it < iters; ++it)
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        if (MODE == 1) {
          tc_fence_after();
          const uint32_t a0 = smem_u32(sm + stage * kStage), b0 = a0 + 16384;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_cg1(tmem, sdesc_sw128(a0 + k * 32, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                     (it | kb | k) ? 1u : 0u);
          commit_cg1(&empty[stage]);
        } else {
          mbar_arrive(&empty[stage]);
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = clock64() - t0;
    out[blockIdx.x * 2 + 1] = (unsigned long long)iters * kblocks * kStage;
  }
  if (MODE == 1 && warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*slot), "r"(256));
  }
}


// Pair mode (mirrors gemm_tc2_kernel's main loop): cluster of 2, each CTA loads A (one 128-row
// box, 16 KB) + B (NB boxes of BR rows = 128 rows, 16 KB) per stage with .cta_group::2 TMA onto
// the LEADER's full barrier; the leader issues 4 cta_group::2 M256 N256 MMAs per stage (512
// cycles ideal) and commits to both CTAs' empty barriers. MMA=false: the leader just releases.
template <int STAGES, int NB, int BR, bool MMA>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe_pair(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int iters,
               unsigned long long* out, int spread) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint32_t* slot = reinterpret_cast<uint32_t*>(empty + STAGES);
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_rank() & 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(slot, 256);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const int pair = blockIdx.x / 2;
  // spread: every pair reads its own A rows and its own B rows (distinct lines, 16 k-blocks
  // per pass over a 38 MB L2-resident region); else 16 row blocks shared by all pairs
  const int r0 = spread ? pair * 256 + rank * 128 : (pair % 16) * 256 + rank * 128;
  const int rb = spread ? (r0 + 9472) % kBigRows : r0;
  const int kblocks = spread ? 16 : kCols / 64;
  const int rep = spread ? iters * (kCols / 64) / 16 : iters;
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < rep; ++it)
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (rank == 0) mbar_expect_tx(&full[stage], 2 * kStage);
        tma_load_2d_pair(&mapA, &full[stage], sm + stage * kStage, kb * 64, r0);
        for (int b = 0; b < NB; ++b)
          tma_load_2d_pair(&mapB, &full[stage], sm + stage * kStage + 16384 + b * BR * 128, kb * 64,
                           rb + b * BR);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
  } else if (threadIdx.x == 32 && rank == 0) {
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t tmem = *slot;
    constexpr uint32_t idesc = idesc_bf16_f32(256, 256, false, false);
    for (int it = 0; it < rep; ++it)
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (MMA) {
          const uint32_t a0 = smem_u32(sm + stage * kStage), b0 = a0 + 16384;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_cg2(tmem, sdesc_sw128(a0 + k * 32, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                          (it | kb | k) ? 1u : 0u);
        }
        umma_commit_cg2_mc(&empty[stage], 0x3);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = clock64() - t0;
    out[blockIdx.x * 2 + 1] = (unsigned long long)rep * kblocks * kStage;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(*slot, 256);
  }
}

struct BigParams {
  CUtensorMap tmA[4], tmB[4], tmD;
  int kbp;
  int pad[200];
};

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    probe_pair_big(const __grid_constant__ BigParams P, int iters, unsigned long long* out) {
  // blockDim 192: warps 2..5 mimic the GEMM epilogue (lane 0 polls a barrier the MMA thread
  // completes at the end); P.pad[0] = TMEM columns to allocate
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint32_t* slot = reinterpret_cast<uint32_t*>(empty + STAGES);
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_rank() & 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  uint64_t* done = reinterpret_cast<uint64_t*>(slot + 2);
  if (threadIdx.x == 0) {
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(slot, P.pad[0]);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const int pair = blockIdx.x / 2;
  const int r0 = (pair % 16) * 256 + rank * 128;
  const int kblocks = P.pad[1] / 64;
  const unsigned long long t0 = clock64();
  if (warp >= 2) {
    if ((threadIdx.x & 31) == 0) mbar_wait(done, 0);
    __syncwarp();
  } else if (threadIdx.x == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it)
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (rank == 0) mbar_expect_tx(&full[stage], 2 * kStage);
        const CUtensorMap* mA = &P.tmA[kb / P.kbp];
        const CUtensorMap* mB = &P.tmB[kb / P.kbp];
        const int kc = (kb % P.kbp) * 64;
        uint8_t* a_dst = P.pad[2] ? sm + stage * 16384 : sm + stage * kStage;
        uint8_t* b_dst = P.pad[2] ? sm + STAGES * 16384 + stage * 16384 : sm + stage * kStage + 16384;
        tma_load_2d_pair(mA, &full[stage], a_dst, kc, r0);
        tma_load_2d_pair(mB, &full[stage], b_dst, kc, r0);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
  } else if (threadIdx.x == 32 && rank == 0) {
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t tmem = *slot;
    constexpr uint32_t idesc = idesc_bf16_f32(256, 256, false, false);
    for (int it = 0; it < iters; ++it)
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a0 = P.pad[2] ? smem_u32(sm + stage * 16384) : smem_u32(sm + stage * kStage);
        const uint32_t b0 = P.pad[2] ? smem_u32(sm + STAGES * 16384 + stage * 16384) : a0 + 16384;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16_cg2(tmem, sdesc_sw128(a0 + k * 32, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                        (it | kb | k) ? 1u : 0u);
        umma_commit_cg2_mc(&empty[stage], 0x3);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
  }
  if (threadIdx.x == 32 || (threadIdx.x == 0 && rank == 1)) mbar_arrive(done);
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = clock64() - t0;
    out[blockIdx.x * 2 + 1] = (unsigned long long)iters * kblocks * kStage;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(*slot, P.pad[0]);
  }
}

__global__ void fill_random(uint16_t* p, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint32_t x = uint32_t(i) * 2654435761u ^ uint32_t(i >> 32);
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    // bf16 in [-1, 1): sign, exponent 120..126, random mantissa
    p[i] = uint16_t(((x & 1) << 15) | ((120 + (x >> 1) % 7) << 7) | ((x >> 8) & 0x7f));
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int STAGES, int NBOX, int ROWS, int MODE>
void run(const char* name, void* src, int grid, int iters) {
  CUtensorMap map;
  cuuint64_t dims[2] = {kCols, kRows};
  cuuint64_t strides[1] = {kCols * 2};
  cuuint32_t box[2] = {64, ROWS};
  cuuint32_t es[2] = {1, 1};
  encode()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = STAGES * NBOX * ROWS * 128 + 1024 + 256;
  auto k = probe<STAGES, NBOX, ROWS, MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* out;
  cudaMalloc(&out, grid * 16);
  k<<<grid, 128, smem>>>(map, 1, out);  // warm L2
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128, smem>>>(map, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(grid * 2);
  cudaMemcpy(h.data(), out, grid * 16, cudaMemcpyDeviceToHost);
  double cyc = 0, bytes = 0;
  for (int i = 0; i < grid; ++i) {
    cyc += h[2 * i];
    bytes += h[2 * i + 1];
  }
  cyc /= grid;
  const cudaError_t err = cudaGetLastError();
  printf("%-28s grid %3d stage %3d KB x%2d  per-SM %6.1f B/clk  chip %6.2f TB/s  clk %5.0f MHz %s\n", name, grid,
         NBOX * ROWS * 128 / 1024, STAGES, bytes / grid / cyc, bytes / (ms * 1e-3) / 1e12, cyc / (ms * 1e3),
         err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
}


template <int STAGES, int NB, int BR, bool MMA>
void run_pair(const char* name, void* src, int grid, int iters, int spread = 0) {
  CUtensorMap mA, mB;
  cuuint64_t dims[2] = {kCols, spread ? kBigRows : kRows};
  cuuint64_t strides[1] = {kCols * 2};
  cuuint32_t boxA[2] = {64, 128}, boxB[2] = {64, BR};
  cuuint32_t es[2] = {1, 1};
  encode()(&mA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  encode()(&mB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = STAGES * 32768 + 1024 + 256;
  auto k = probe_pair<STAGES, NB, BR, MMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* out;
  cudaMalloc(&out, grid * 16);
  k<<<grid, 128, smem>>>(mA, mB, 1, out, spread);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128, smem>>>(mA, mB, iters, out, spread);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(grid * 2);
  cudaMemcpy(h.data(), out, grid * 16, cudaMemcpyDeviceToHost);
  double cyc = 0, bytes = 0;
  for (int i = 0; i < grid; ++i) {
    cyc += h[2 * i];
    bytes += h[2 * i + 1];
  }
  cyc /= grid;
  const double stages = bytes / grid / 32768;
  const cudaError_t err = cudaGetLastError();
  printf("%-28s grid %3d x%d stages  per-SM %6.1f B/clk  %6.0f cyc/stage (MMA floor 512)  clk %5.0f MHz %s\n", name,
         grid, STAGES, bytes / grid / cyc, cyc / stages, cyc / (ms * 1e3), err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
}

void run_big(const char* name, void* src, int grid, int iters, int panels, int threads = 128, int tmem = 256,
             int extra_smem = 0, int pitch = kCols, int split_layout = 0) {
  BigParams P{};
  P.pad[0] = tmem;
  P.pad[1] = pitch;
  P.pad[2] = split_layout;
  cuuint64_t dims[2] = {(cuuint64_t)(pitch / panels), (cuuint64_t)kRows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  for (int p = 0; p < panels; ++p) {
    encode()(&P.tmA[p], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (char*)src + p * (pitch / panels) * 2, dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    P.tmB[p] = P.tmA[p];
  }
  P.kbp = pitch / 64 / panels;
  const int smem = 6 * 32768 + 1024 + 256 + extra_smem;
  auto k = probe_pair_big<6>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* out;
  cudaMalloc(&out, grid * 16);
  k<<<grid, threads, smem>>>(P, 1, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, threads, smem>>>(P, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(grid * 2);
  cudaMemcpy(h.data(), out, grid * 16, cudaMemcpyDeviceToHost);
  double cyc = 0, bytes = 0;
  for (int i = 0; i < grid; ++i) {
    cyc += h[2 * i];
    bytes += h[2 * i + 1];
  }
  cyc /= grid;
  const cudaError_t err = cudaGetLastError();
  printf("%-28s grid %3d  per-SM %6.1f B/clk  %6.0f cyc/stage  clk %5.0f MHz %s\n", name, grid, bytes / grid / cyc,
         cyc / (bytes / grid / 32768), cyc / (ms * 1e3), err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
}

// Persistent-unit variant: units of UNIT k-blocks, TMEM accumulator double-buffered, the leader
// commits tfull per unit, epilogue warps 2..5 (both CTAs) wait tfull and arrive on the leader's
// tempty (count 8), the MMA thread waits tempty before reusing an accumulator: the GEMM's control.
template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    probe_units(const __grid_constant__ BigParams P, int units, int unit_kb, unsigned long long* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int kStage = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const int pair = blockIdx.x / 2;
  const int r0 = (pair % 16) * 256 + rank * 128;
  const int kblocks = P.pad[1] / 64;
  const unsigned long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = 0; u < units; ++u)
        for (int j = 0; j < unit_kb; ++j) {
          const int kb = (u * unit_kb + j) % kblocks;
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * kStage);
          tma_load_2d_pair(&P.tmA[0], &full[stage], sm + stage * 16384, kb * 64, r0);
          tma_load_2d_pair(&P.tmB[0], &full[stage], sm + STAGES * 16384 + stage * 16384, kb * 64, r0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      constexpr uint32_t idesc = idesc_bf16_f32(256, 256, false, false);
      for (int u = 0; u < units; ++u) {
        mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * 256;
        for (int j = 0; j < unit_kb; ++j) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sm + stage * 16384), b0 = smem_u32(sm + STAGES * 16384 + stage * 16384);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_cg2(d, sdesc_sw128(a0 + k * 32, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                          (j | k) ? 1u : 0u);
          umma_commit_cg2_mc(&empty[stage], 0x3);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_cg2_mc(&tfull[acc], 0x3);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t lead = crank & ~1u;
    for (int u = 0; u < units; ++u) {
      if (lane == 0) mbar_wait(&tfull[acc], acc_phase);
      __syncwarp();
      tc_fence_after();
      if (P.pad[3]) {  // read the accumulator rows of this warp like the epilogue does
        uint32_t r[32];
        const uint32_t t_row = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + acc * 256;
        float sum = 0.f;
        for (int c = 0; c < 256; c += 32) {
          tmem_ld32(t_row + c, r);
          tmem_wait_ld();
          for (int i = 0; i < 32; ++i) sum += __uint_as_float(r[i]);
        }
        if (sum == 12345.f) out[0] = 1;  // keep the loads
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[acc], lead);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = clock64() - t0;
    out[blockIdx.x * 2 + 1] = (unsigned long long)units * unit_kb * kStage;
  }
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem, 512);
  }
}

void run_units(const char* name, void* src, int grid, int units, int unit_kb, int epi_ld) {
  BigParams P{};
  P.pad[1] = 4096;
  P.pad[3] = epi_ld;
  cuuint64_t dims[2] = {4096, (cuuint64_t)kRows};
  cuuint64_t strides[1] = {4096 * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  encode()(&P.tmA[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  encode()(&P.tmB[0], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (char*)src + size_t(kRows) * 4096 * 2, dims, strides, box,
           es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 6 * 32768 + 32768 + 1024 + 256;
  auto k = probe_units<6>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* out;
  cudaMalloc(&out, grid * 16);
  k<<<grid, 192, smem>>>(P, 2, unit_kb, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 192, smem>>>(P, units, unit_kb, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(grid * 2);
  cudaMemcpy(h.data(), out, grid * 16, cudaMemcpyDeviceToHost);
  double cyc = 0, bytes = 0;
  for (int i = 0; i < grid; ++i) {
    cyc += h[2 * i];
    bytes += h[2 * i + 1];
  }
  cyc /= grid;
  const cudaError_t err = cudaGetLastError();
  printf("%-28s grid %3d  %6.0f cyc/stage  clk %5.0f MHz %s\n", name, grid, cyc / (bytes / grid / 32768),
         cyc / (ms * 1e3), err == cudaSuccess ? "" : cudaGetErrorString(err));
  cudaFree(out);
}

int main() {
  void* src;
  cudaMalloc(&src, size_t(kBigRows) * kCols * 2);
  cudaMemset(src, 0, size_t(kBigRows) * kCols * 2);
  if (getenv("RANDOM")) fill_random<<<1184, 256>>>(reinterpret_cast<uint16_t*>(src), size_t(kBigRows) * kCols);
  if (getenv("UNITS_ONLY")) {
    for (int grid : {64, 148}) {
      run_units("units 64kb no-epi-ld", src, grid, 16, 64, 0);
      run_units("units 64kb epi-ld", src, grid, 16, 64, 1);
      run_units("units 1024kb no-epi-ld", src, grid, 1, 1024, 0);
    }
    return 0;
  }
  if (getenv("BIG_ONLY")) goto big;
  for (int grid : {16, 74, 148}) {
    run_pair<6, 1, 128, false>("spread pair fill", src, grid, 8, 1);
    run_pair<6, 1, 128, true>("spread pair mma", src, grid, 8, 1);
  }
  for (int grid : {16, 148}) {
    run_pair<6, 1, 128, false>("pair fill B 1x128", src, grid, 8);
    run_pair<6, 2, 64, false>("pair fill B 2x64", src, grid, 8);
    run_pair<6, 1, 128, true>("pair mma B 1x128", src, grid, 8);
    run_pair<6, 2, 64, true>("pair mma B 2x64", src, grid, 8);
  }
  if (getenv("PAIR_ONLY")) return 0;
big:
  if (getenv("BIG_ONLY")) {
    for (int grid : {16, 148}) {
      run_big("interleaved stages", src, grid, 16, 1, 192, 512, 32768, 4096, 0);
      run_big("A stages | B stages", src, grid, 16, 1, 192, 512, 32768, 4096, 1);
    }
    return 0;
  }
  for (int grid : {16, 74, 148}) {
    run<6, 1, 128, 0>("fill 1x128rows", src, grid, 8);
    run<6, 2, 128, 0>("fill 2x128rows", src, grid, 8);
    run<6, 1, 256, 0>("fill 1x256rows", src, grid, 8);
    run<12, 1, 128, 0>("fill 1x128rows deep", src, grid, 8);
    run<4, 3, 128, 0>("fill 3x128rows", src, grid, 8);
    run<4, 3, 128, 1>("mma N256 + fill 3x128", src, grid, 8);
  }
  return 0;
}
