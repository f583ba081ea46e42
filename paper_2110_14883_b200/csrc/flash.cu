// Fused attention forward for sm_100a: O = softmax(Q K^T scale) V per problem (batch x head),
// the scores never leaving the SM (online softmax over key tiles; the two-pass form of rsa.cu
// writes every score to HBM and reads it back). Used by the attention core (attn.cu) for the
// local problems of every TP layout. bf16 in, fp32 accumulation and statistics, bf16 out.
//
// One CTA per (problem, 128-query tile); 192 threads:
//   warp 0    TMA: Q once, then K / V tiles of 128 keys through a 2-stage ring;
//   warp 1    tcgen05 MMA issuer (cta_group::1): S_j = Q K_j^T into one of two TMEM score
//             buffers (128 columns each), O += P_j V_j into the TMEM output accumulator;
//   warps 2-5 softmax (one query row per thread, TMEM lane quadrant = warp % 4): row max of
//             S_j, p = exp2(s * scale log2 e - m), running sum, bf16 P_j to shared memory in
//             the 128-byte-swizzled K-major layout the PV MMA reads, and the rescale of the O row
//             by exp2(m_old - m_new) (tcgen05.ld / st) before P_j V_j is accumulated.
// Keys past the sequence end are masked to -inf (their K / V rows are read but weigh 0).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <mutex>

#include "sm100_ptx.cuh"
#include "tp_internal.h"

namespace tp {
volatile unsigned* g_flash_dbg = nullptr;  // tools only (tp_flash_debug)
namespace {

using namespace ptx;

// Softmax warps: 4 (one per TMEM lane quadrant, all 128 keys of a row) or 8 (two per
// quadrant, each 64 keys of the row and half of O's columns; the row max is exchanged through
// shared memory, the row sums are combined at the end). 8 for d = 64, whose tiles are bound
// by the exp2 stream (the XU pipe) rather than the tensor core; d = 128 has no smem left for
// the exchange and is balanced.
#ifndef TP_FLASH_W128
#define TP_FLASH_W128 0  // d = 128 with eight softmax warps + one P buffer: measured slower (profiles/r01_exp51_w128.log)
#endif
template <int D>
constexpr int soft_warps();
// d = 64 as two CTAs per SM (TP_FLASH_2CTA64): 4 softmax warps, one S and one P buffer, one K/V
// stage, 256 TMEM columns and FC<64>::Smem = 83,200 B of shared memory each (Q 16 KB + K/V
// 32 KB + P 32 KB + barriers), so two query tiles share an SM and one CTA's softmax overlaps the
// other's MMAs
#ifndef TP_FLASH_KV64
#define TP_FLASH_KV64 2  // K / V ring depth for d = 64 (3 measured equal: profiles/r01_exp58_kv64.log)
#endif
#ifndef TP_FLASH_2CTA64
#define TP_FLASH_2CTA64 1
#endif
template <int D>
constexpr bool two_cta() { return D == 64 && TP_FLASH_2CTA64; }
template <int D>
constexpr int kv_stages() { return two_cta<D>() ? 1 : (D == 64 ? TP_FLASH_KV64 : 2); }
template <int D>
constexpr int soft_warps() { return TP_FLASH_W128 && D == 128 ? 8 : (D == 64 ? (two_cta<D>() ? 4 : 8) : 4); }
// P buffers in shared memory: two (the softmax runs a tile ahead of P V), one for d = 128 with
// eight softmax warps (no shared memory left for a second buffer and the max exchange)
template <int D>
constexpr int p_bufs() { return (D == 128 && soft_warps<D>() == 8) || two_cta<D>() ? 1 : 2; }
template <int D>
constexpr int f_threads() { return 64 + 32 * soft_warps<D>(); }
constexpr int kQT = 128;   // query rows per CTA
constexpr int kKT = 128;   // keys per tile
template <int D>
constexpr int kv_stages();
// S_j = Q K_j^T buffers in TMEM (2; 3 measured equal: profiles/r01_exp50_sbuf.log). Three let S run two tiles ahead of P V (S_{j+2}
// is queued right after P_{j-1} V_{j-1}), so the softmax never waits for its scores; with O
// that is 3 x 128 + D <= 512 columns for D <= 128.
#ifndef TP_FLASH_SBUF
#define TP_FLASH_SBUF 2
#endif
constexpr int kSBuf = TP_FLASH_SBUF;
template <int D>
constexpr int s_bufs() { return two_cta<D>() ? 1 : kSBuf; }
template <int D>
constexpr int tmem_cols_of() { return two_cta<D>() ? 256 : 512; }

template <int D>
struct FC {
  static constexpr int QBytes = kQT * D * 2;           // D/64 boxes of [128 rows][128 B]
  static constexpr int KBytes = kKT * D * 2;
  static constexpr int VBytes = kKT * D * 2;           // 2 key blocks x D/64 chunks of [64][128 B]
  static constexpr int PBytes = kQT * kKT * 2;         // 2 key blocks of [128 rows][128 B]
  static constexpr int StageBytes = KBytes + VBytes;
  static constexpr int XBytes = soft_warps<D>() == 8 ? 2 * 2 * kQT * 4 : 0;  // [tile parity][half][row]
  static constexpr int Smem = QBytes + kv_stages<D>() * StageBytes + p_bufs<D>() * PBytes + XBytes + 1024 + 256;
};

struct FParams {
  CUtensorMap tmQ, tmK, tmV;
  __nv_bfloat16* out;
  int64_t s, problems;
  float scale_log2;  // scale * log2(e)
  volatile unsigned* dbg;  // tools only: progress markers (mapped host memory) or null
  // Carried online softmax (ring attention: one call per K / V block of the ring). acc
  // [problems*s, D] fp32 holds the unnormalised O of the blocks seen so far and ml
  // [problems*s, 2] fp32 their row max (scaled log2 units) and row sum. carry_in: start
  // from (acc, ml) instead of empty; last: write O / l to `out` (bf16), else (acc, ml).
  float* acc;
  float* ml;
  int carry_in, last;
  // optional: per-row log-sum-exp in scaled log2 units, lse = m + log2(l), so that the
  // probabilities are exp2(s scale log2e - lse) (the fused backward recomputes them)
  float* lse;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (Cody-Waite split x = n + f, |f| <= 1/2, degree-4 Taylor of 2^f, relative
// error < 5e-5, below bf16's 4e-3): takes part of the exponentials off the XU pipe (16 / clk / SM)
// that bounds the softmax. x >= -126 (masked keys give 2^-126 ~ 1e-38, not 0: negligible).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: the integer part lands in the low mantissa bits
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.0096181291f, 0.0555041087f);
  p = fmaf(p, f, 0.2402265070f);
  p = fmaf(p, f, 0.6931471806f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
#ifndef TP_FLASH_POLY_EVERY
#define TP_FLASH_POLY_EVERY 0  // one exp pair in every N on the FMA pipe; 0 = none (measured: no gain, the softmax is latency-bound, profiles/r01_exp49_poly_exp.log)
#endif

template <int D>
__global__ void __launch_bounds__(f_threads<D>(), two_cta<D>() ? 2 : 1) flash_fwd_kernel(const __grid_constant__ FParams F) {
  constexpr int SB = s_bufs<D>();
  using C = FC<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = sQ + C::QBytes;
  uint8_t* sP = sKV + kv_stages<D>() * C::StageBytes;
  constexpr int NP = p_bufs<D>();
  float* sX = reinterpret_cast<float*>(sP + NP * C::PBytes);  // P buffers; max exchange
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + NP * C::PBytes + C::XBytes);
  uint64_t* q_full = bars;
  // K and V have their own barriers: K_j's slot frees when S_j retires (early), V_j's when
  // P_j V_j retires, so K_{j+2}'s load is in flight long before S_{j+2} is issued
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + kv_stages<D>();
  uint64_t* v_full = k_empty + kv_stages<D>();
  uint64_t* v_empty = v_full + kv_stages<D>();
  uint64_t* s_full = v_empty + kv_stages<D>();
  uint64_t* s_empty = s_full + SB;
  uint64_t* p_full = s_empty + SB;   // [2] P_j in buffer j % 2 written (and O rescaled)
  uint64_t* p_empty = p_full + 2;   // [2] P_j V_j retired: P buffer j % 2 free, O up to date
  uint32_t* tslot = reinterpret_cast<uint32_t*>(p_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t prob = blockIdx.y;
  const int64_t q0 = int64_t(blockIdx.x) * kQT;
  const int64_t row_base = prob * F.s;          // first row of this problem in [problems*s, D]
  const int ntiles = static_cast<int>((F.s + kKT - 1) / kKT);

  if (threadIdx.x == 0) {
    tma_prefetch(&F.tmQ);
    tma_prefetch(&F.tmK);
    tma_prefetch(&F.tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < kv_stages<D>(); ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < SB; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], soft_warps<D>());
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], soft_warps<D>());
      mbar_init(&p_empty[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg1(tslot, tmem_cols_of<D>());
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  auto tS = [&](int b) { return tmem + static_cast<uint32_t>(b * kKT); };
  const uint32_t tO = tmem + SB * kKT;

  if (warp == 0) {
    if (elect_one()) {
      // ---- TMA producer
      mbar_expect_tx(q_full, C::QBytes);
      for (int c = 0; c < D / 64; ++c)
        tma_load_2d(&F.tmQ, q_full, sQ + c * kQT * 128, c * 64, static_cast<int>(row_base + q0));
      auto load_k = [&](int j) {
        const int st = j % kv_stages<D>();
        mbar_wait(&k_empty[st], ((j / kv_stages<D>()) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], C::KBytes);
        uint8_t* kd = sKV + st * C::StageBytes;
        const int key0 = static_cast<int>(row_base + int64_t(j) * kKT);
        for (int c = 0; c < D / 64; ++c) tma_load_2d(&F.tmK, &k_full[st], kd + c * kKT * 128, c * 64, key0);
      };
      auto load_v = [&](int j) {
        const int st = j % kv_stages<D>();
        mbar_wait(&v_empty[st], ((j / kv_stages<D>()) & 1) ^ 1);
        mbar_expect_tx(&v_full[st], C::VBytes);
        uint8_t* vd = sKV + st * C::StageBytes + C::KBytes;
        const int key0 = static_cast<int>(row_base + int64_t(j) * kKT);
        // V: MN-major B operand, per 64-key block the D/64 chunks of [64 keys][64 d]
        for (int kb = 0; kb < 2; ++kb)
          for (int c = 0; c < D / 64; ++c)
            tma_load_2d(&F.tmV, &v_full[st], vd + (kb * (D / 64) + c) * 64 * 128, c * 64, key0 + kb * 64);
      };
      // K runs one tile ahead of V (S_{j+1} is issued before P_j V_j)
      for (int j = 0; j < SB - 1 && j < ntiles; ++j) load_k(j);
      for (int j = 0; j < ntiles; ++j) {
        if (F.dbg && blockIdx.x == 0 && blockIdx.y == 0) F.dbg[0] = 100 + j;
        if (j + SB - 1 < ntiles) load_k(j + SB - 1);
        load_v(j);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      // ---- MMA issuer
      constexpr uint32_t idS = idesc_bf16_f32(128, kKT, false, false);
      constexpr uint32_t idO = idesc_bf16_f32(128, D, false, true);
      const uint64_t qd = sdesc_sw128(smem_u32(sQ), 16, 1024);
      auto issue_s = [&](int j) {
        const int st = j % kv_stages<D>();
        mbar_wait(&k_full[st], (j / kv_stages<D>()) & 1);
        if (F.dbg && blockIdx.x == 0 && blockIdx.y == 0) F.dbg[1] = 200 + j;
        const int b = j % SB;
        mbar_wait(&s_empty[b], ((j / SB) & 1) ^ 1);  // softmax done with S_{j-SB}
        if (F.dbg && blockIdx.x == 0 && blockIdx.y == 0) F.dbg[2] = 300 + j;
        tc_fence_after();
        const uint64_t kdsc = sdesc_sw128(smem_u32(sKV + st * C::StageBytes), 16, 1024);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          // K step of 16 inside a 64-wide box: +32 B; next box: +128 rows x 128 B
          const uint32_t off = (k / 4) * (kQT * 128 / 16) + (k % 4) * 2;
          const uint32_t offk = (k / 4) * (kKT * 128 / 16) + (k % 4) * 2;
          umma_bf16_cg1(tS(b), qd + off, kdsc + offk, idS, k > 0 ? 1u : 0u);
        }
        umma_commit_cg1(&s_full[b]);
        umma_commit_cg1(&k_empty[st]);  // K_j read
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < SB - 1 && j < ntiles; ++j) issue_s(j);
      for (int j = 0; j < ntiles; ++j) {
        if (j + SB - 1 < ntiles) issue_s(j + SB - 1);
        if (F.dbg && blockIdx.x == 0 && blockIdx.y == 0) F.dbg[3] = 400 + j;
        const int pb = j % NP;
        mbar_wait(&p_full[pb], (j / NP) & 1);  // P_j in smem, O rescaled
        if (F.dbg && blockIdx.x == 0 && blockIdx.y == 0) F.dbg[4] = 500 + j;
        tc_fence_after();
        const int st = j % kv_stages<D>();
        mbar_wait(&v_full[st], (j / kv_stages<D>()) & 1);
        tc_fence_after();
        const uint64_t pd = sdesc_sw128(smem_u32(sP + pb * C::PBytes), 16, 1024);
        const uint64_t vdsc = sdesc_sw128(smem_u32(sKV + st * C::StageBytes + C::KBytes), 64 * 128, 1024);
#pragma unroll
        for (int k = 0; k < kKT / 16; ++k) {
          const int kb = k / 4, kk = k % 4;
          const uint32_t offp = kb * (kQT * 128 / 16) + kk * 2;                 // K-major P
          const uint32_t offv = kb * ((D / 64) * 64 * 128 / 16) + kk * (2048 / 16);  // MN-major V
          umma_bf16_cg1(tO, pd + offp, vdsc + offv, idO, (j > 0 || k > 0 || F.carry_in) ? 1u : 0u);
        }
        umma_commit_cg1(&v_empty[st]);
        umma_commit_cg1(&p_empty[pb]);
      }
    }
    __syncwarp();
  } else {
    // ---- softmax warps: row = (warp % 4) * 32 + lane; with 8 warps the two warps of a lane
    // quadrant take keys [half * 64, +64) of every tile and O columns [half * D/2, +D/2)
    constexpr int kH = soft_warps<D>() / 4;  // warps per quadrant
    constexpr int KW = kKT / kH;             // keys per warp per tile
    constexpr int OC = D / kH;               // O columns per warp
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t s_off = static_cast<uint32_t>(half * KW);
    const uint32_t o_off = static_cast<uint32_t>(half * OC);
    float m = -INFINITY, l = 0.f;  // l: this warp's keys only (the halves are added at the end)
    const int64_t qrow = q0 + r;  // this thread's query row within the problem
    if (F.carry_in && qrow < F.s) {
      const float2 c = *reinterpret_cast<const float2*>(F.ml + 2 * (row_base + qrow));
      m = c.x;
      l = half == 0 ? c.y : 0.f;
    }
    for (int j = 0; j < ntiles; ++j) {
      const int b = j % SB;
      mbar_wait(&s_full[b], (j / SB) & 1);
      tc_fence_after();
      const int64_t valid = F.s - int64_t(j) * kKT - half * KW;  // this warp's keys in range
      // this warp's part of the S row into registers once: all loads in flight, one wait
      uint32_t sv[KW / 32][32];
#pragma unroll
      for (int c = 0; c < KW / 32; ++c) tmem_ld32(tS(b) + lane_off + s_off + c * 32, sv[c]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[b]);  // S buffer b may be overwritten
      if (valid < KW) {  // last tile of a ragged sequence: masked keys weigh exp2(-inf) = 0
#pragma unroll
        for (int c = 0; c < KW / 32; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i >= valid) sv[c][i] = 0xff800000u;  // -inf
      }
      auto sval = [&](int c, int i) { return __uint_as_float(sv[c][i]); };
      // row max: 8 independent chains, then a tree (a single long fmax chain is latency)
      float mxs[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mxs[i] = -INFINITY;
#pragma unroll
      for (int c = 0; c < KW / 32; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) mxs[i & 7] = fmaxf(mxs[i & 7], sval(c, i));
      float mx = fmaxf(fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3])),
                       fmaxf(fmaxf(mxs[4], mxs[5]), fmaxf(mxs[6], mxs[7])));
      if (kH == 2) {  // the other half's max of the same row (double-buffered by tile parity)
        const uint32_t xc = smem_u32(sX) + (j & 1) * (2 * kQT * 4);
        sts32(xc + (half * kQT + r) * 4, mx);
        named_barrier_sync(1 + quad, 64);
        mx = fmaxf(mx, lds32(xc + ((half ^ 1) * kQT + r) * 4));
      }
      // Lazy rescale: the reference max m moves only when some row of the warp would exceed it
      // by more than 2^8 (p <= 256 is exact enough in bf16 / fp32), so most tiles leave O alone
      // and the softmax runs a tile ahead of the P V MMA. O, l and the carried (m, l) all use
      // the same reference, so O / l is unchanged. Both warps of a quadrant see the same rows
      // and the same row max, so they take the same decision.
      const float m_cand = fmaxf(m, mx * F.scale_log2);
      const bool move = (j == 0 && !F.carry_in) || __any_sync(0xffffffffu, m_cand > m + 8.f);
      const float m_new = move ? m_cand : m;
      const float alpha = exp2f(m - m_new);  // 1 when m stays; 0 on the first tile (m = -inf)
      // P buffer j % NP was last read by P_{j-NP} V_{j-NP}
      if (j >= NP) mbar_wait(&p_empty[j % NP], ((j - NP) / NP) & 1);
      tc_fence_after();
      // p = exp2(s scale log2e - m_new) (one FFMA + MUFU.EX2 each) -> bf16 P row (swizzled
      // K-major), row sum in 8 independent partial sums
      float rsp[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rsp[i] = 0.f;
      const float neg_m = -m_new;
#pragma unroll
      for (int c = 0; c < KW / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const bool poly = TP_FLASH_POLY_EVERY > 0 && (i % (TP_FLASH_POLY_EVERY > 0 ? TP_FLASH_POLY_EVERY : 1)) ==
                                                          (TP_FLASH_POLY_EVERY > 0 ? TP_FLASH_POLY_EVERY - 1 : 0);
          const float x0 = fmaf(sval(c, 2 * i), F.scale_log2, neg_m);
          const float x1 = fmaf(sval(c, 2 * i + 1), F.scale_log2, neg_m);
          const float p0 = poly ? ex2_poly(x0) : ex2_approx(x0);
          const float p1 = poly ? ex2_poly(x1) : ex2_approx(x1);
          rsp[i & 7] += p0 + p1;
          __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
          pk[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        // 32 keys = 64 B = 4 swizzled 16-byte chunks of the row in key block (key / 64)
        const int key0 = half * KW + c * 32;
        const uint32_t rowp = smem_u32(sP) + (j % NP) * C::PBytes + (key0 / 64) * (kQT * 128) + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = ((key0 % 64) / 32) * 4 + q;
          sts128(rowp + ((chunk ^ (r & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      const float rs = ((rsp[0] + rsp[1]) + (rsp[2] + rsp[3])) + ((rsp[4] + rsp[5]) + (rsp[6] + rsp[7]));
      l = l * alpha + rs;
      if (j == 0 && F.carry_in) {
        // carried O of the earlier ring blocks, rescaled to this block's running max, into
        // TMEM before the first P V MMA accumulates onto it
        const float4* src = reinterpret_cast<const float4*>(F.acc + (row_base + qrow) * D + o_off);
#pragma unroll 1
        for (int c = 0; c < OC / 32; ++c) {
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 x = qrow < F.s ? src[c * 8 + i] : make_float4(0.f, 0.f, 0.f, 0.f);
            v[4 * i] = __float_as_uint(x.x * alpha);
            v[4 * i + 1] = __float_as_uint(x.y * alpha);
            v[4 * i + 2] = __float_as_uint(x.z * alpha);
            v[4 * i + 3] = __float_as_uint(x.w * alpha);
          }
          tmem_st32(tO + lane_off + o_off + c * 32, v);
        }
        tmem_wait_st();
      }
      // rescale this warp's O columns (warp-uniform: tcgen05.ld / st are .sync.aligned)
      if (j > 0 && move) {
        mbar_wait(&p_empty[(j - 1) % NP], ((j - 1) / NP) & 1);  // P_{j-1} V_{j-1} retired
        tc_fence_after();
        uint32_t v[OC / 32][32];
#pragma unroll
        for (int c = 0; c < OC / 32; ++c) tmem_ld32(tO + lane_off + o_off + c * 32, v[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < OC / 32; ++c) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[c][i] = __float_as_uint(__uint_as_float(v[c][i]) * alpha);
          tmem_st32(tO + lane_off + o_off + c * 32, v[c]);
        }
        tmem_wait_st();
      }
      m = m_new;
      fence_proxy_async_smem();  // P visible to the MMA (async proxy)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j % NP]);
    }
    // epilogue: O / l -> bf16 row (this warp's columns)
    mbar_wait(&p_empty[(ntiles - 1) % NP], ((ntiles - 1) / NP) & 1);
    tc_fence_after();
    if (kH == 2) {  // full row sum = the two halves' sums
      const uint32_t xc = smem_u32(sX) + (ntiles & 1) * (2 * kQT * 4);  // parity the last tile did not use
      sts32(xc + (half * kQT + r) * 4, l);
      named_barrier_sync(1 + quad, 64);
      l += lds32(xc + ((half ^ 1) * kQT + r) * 4);
    }
    const int64_t q = q0 + r;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    if (F.last && F.lse && half == 0 && q < F.s) F.lse[row_base + q] = m + __log2f(l);
    if (!F.last) {  // carry out: unnormalised O (fp32) and (m, l) for the next ring block
#pragma unroll 1
      for (int c = 0; c < OC / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tO + lane_off + o_off + c * 32, v);
        tmem_wait_ld();
        if (q < F.s) {
          float4* dst = reinterpret_cast<float4*>(F.acc + (row_base + q) * D + o_off + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                 __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        }
      }
      if (q < F.s && half == 0) *reinterpret_cast<float2*>(F.ml + 2 * (row_base + q)) = make_float2(m, l);
    }
#pragma unroll 1
    for (int c = 0; c < (F.last ? OC / 32 : 0); ++c) {
      uint32_t v[32];
      tmem_ld32(tO + lane_off + o_off + c * 32, v);
      tmem_wait_ld();
      if (q < F.s) {
        __nv_bfloat16* dst = F.out + (row_base + q) * D + o_off + c * 32;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 u;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            h[k] = __floats2bfloat162_rn(__uint_as_float(v[i + 2 * k]) * inv, __uint_as_float(v[i + 2 * k + 1]) * inv);
          *reinterpret_cast<uint4*>(dst + i) = u;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg1(tmem, tmem_cols_of<D>());
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

tp_status map(CUtensorMap* m, const void* base, uint64_t rows, int D, uint32_t box_rows) {
  auto fn = encode();
  if (!fn) return fail(TP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), rows};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(TP_ERR_SHAPE, "flash: tensor map encode failed");
  return TP_OK;
}

template <int D>
tp_status launch(const FParams& F, cudaStream_t s) {
  using C = FC<D>;
  auto k = flash_fwd_kernel<D>;
  TP_CUDA(set_smem_attr(reinterpret_cast<const void*>(k), C::Smem));
  dim3 grid(static_cast<unsigned>((F.s + kQT - 1) / kQT), static_cast<unsigned>(F.problems));
  k<<<grid, f_threads<D>(), C::Smem, s>>>(F);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace

bool flash_supported(int64_t d, tp_dtype dt) { return dt == TP_BF16 && (d == 64 || d == 128); }

// q, k, v, out: [problems, s, d] bf16 contiguous.
tp_status flash_attn_fwd(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                         const void* v, void* out, float scale, cudaStream_t st, float* lse) {
  if (!problems || !s) return TP_OK;
  if (d != 64 && d != 128) return fail(TP_ERR_UNSUPPORTED, "flash: d must be 64 or 128");
  if (problems > 65535) return fail(TP_ERR_UNSUPPORTED, "flash: too many problems for one grid");
  FParams F{};
  const uint64_t rows = uint64_t(problems) * uint64_t(s);
  TP_TRY(map(&F.tmQ, q, rows, static_cast<int>(d), kQT));
  TP_TRY(map(&F.tmK, k, rows, static_cast<int>(d), kKT));
  TP_TRY(map(&F.tmV, v, rows, static_cast<int>(d), 64));
  F.out = static_cast<__nv_bfloat16*>(out);
  F.s = s;
  F.problems = problems;
  F.scale_log2 = scale * 1.4426950408889634f;
  F.dbg = g_flash_dbg;
  F.last = 1;
  F.lse = lse;
  return d == 64 ? launch<64>(F, st) : launch<128>(F, st);
}

// One block of a ring: q [problems, s, d]; k, v [problems, s, d] (this ring step's block);
// acc [problems*s, d] fp32 and ml [problems*s, 2] fp32 carry the online softmax between calls.
tp_status flash_attn_fwd_carry(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                               const void* v, void* out, float* acc, float* ml, bool carry_in,
                               bool last, float scale, cudaStream_t st, float* lse) {
  if (!problems || !s) return TP_OK;
  if (d != 64 && d != 128) return fail(TP_ERR_UNSUPPORTED, "flash: d must be 64 or 128");
  if (problems > 65535) return fail(TP_ERR_UNSUPPORTED, "flash: too many problems for one grid");
  if (!acc || !ml) return fail(TP_ERR_ARG, "flash: carry buffers are null");
  FParams F{};
  const uint64_t rows = uint64_t(problems) * uint64_t(s);
  TP_TRY(map(&F.tmQ, q, rows, static_cast<int>(d), kQT));
  TP_TRY(map(&F.tmK, k, rows, static_cast<int>(d), kKT));
  TP_TRY(map(&F.tmV, v, rows, static_cast<int>(d), 64));
  F.out = static_cast<__nv_bfloat16*>(out);
  F.s = s;
  F.problems = problems;
  F.scale_log2 = scale * 1.4426950408889634f;
  F.dbg = g_flash_dbg;
  F.acc = acc;
  F.ml = ml;
  F.carry_in = carry_in ? 1 : 0;
  F.last = last ? 1 : 0;
  F.lse = last ? lse : nullptr;
  return d == 64 ? launch<64>(F, st) : launch<128>(F, st);
}

}  // namespace tp
