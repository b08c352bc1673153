// mlp_tc.cu -- the per-step policy forward (a1; tanh hidden and output, R13/R14)
// of WIDE policies (C3: 4-256-256-256-1) on the 5th-generation tensor cores.
//
// One CTA owns 128 trajectories and runs every layer for them:
//   D[128 x out] = H[128 x in] . W_l^T  on tcgen05 (kind::f16, fp32 TMEM accumulator), with the same
//   3-pass fp16 split as the GP contraction (h = h_hi + h_lo, W = W_hi + W_lo;
//   h.W ~ h_hi W_hi + h_hi W_lo + h_lo W_hi, fp32-class accuracy, tests/test_gpu_tc.py),
//   then bias + tanh in the epilogue, which also writes the activation tape and places the next
//   layer's input H (hi | lo, fp16 pairs) straight into TMEM as the A operand of the next layer's
//   TS-form MMAs.  The weights are packed once per rollout (k_pack_mlp) into K-chunks of the
//   canonical no-swizzle K-major layout (tc.cuh), streamed by 1-D bulk copies through a 3-stage
//   ring.  TMEM: accumulator columns [0, 256), H hi [256, 384), H lo [384, 512).
// Warps 0-15: epilogue (warp w: TMEM lane quarter w % 4, column group w / 4); warp 16: weight
// producer; warp 17: MMA issuer.  Replaces the register-tiled fp32 GEMM k_mlp_fwd (mlp_tiled.cu),
// which is shared-memory-latency bound at 8 warps per SM.
#include <cuda_fp16.h>
#include <stdlib.h>

#include <algorithm>

#include "bagel_internal.h"
#include "tc.cuh"

namespace mtc {

constexpr int ROWS = 128;
constexpr int KCH = 64;          // K elements per pipeline stage
constexpr int NST = 2;           // ring stages
constexpr int WB_LD = 20;        // per-warp store staging: 32 rows x 16 columns, rows padded to 20 floats
constexpr int EPI_WARPS = 16;    // 4 per TMEM lane quarter, each a quarter of the columns
constexpr int THREADS = 32 * (EPI_WARPS + 2);
constexpr int MAXCH = 32;        // chunks over all layers (8 layers x 4 chunks of 64)
constexpr uint32_t ACC = 0, AHI = 256, ALO = 384;
constexpr size_t STAGE_BYTES = (size_t)BAGEL_MAX_WIDTH * KCH * 2 * 2;  // hi + lo of 256 x 64 fp16

struct Args {
  PolicyDesc P;
  int p, D, B;
  const uint8_t* wpk;            // packed weight chunks
  int nch;
  int ch_layer[MAXCH], ch_k0[MAXCH], ch_kc[MAXCH];
  long long ch_off[MAXCH];
  int Np[BAGEL_MAX_LAYERS];      // out rounded up to 16 (>= 16)
  const float* theta;            // biases
  const float* x;                // B x p (this step's state)
  const float* goals;            // B x p
  float* act;                    // B x act_ld (this step's activation tape rows)
  float* xstar;                  // B x D
};

inline int rup(int a, int b) { return (a + b - 1) / b * b; }

// Chunk table of a policy (host): chunk q of layer l covers K elements [k0, k0 + kc) (kc a multiple
// of 16), packed as [hi: Np x kc | lo: Np x kc] fp16 canonical K-major (KT = kc).
void chunk_table(const PolicyDesc& P, Args& a, size_t* total) {
  size_t off = 0;
  a.nch = 0;
  for (int l = 0; l < P.n_layers; ++l) {
    const int Kp = rup(P.sizes[l], 16), Np = std::max(16, rup(P.sizes[l + 1], 16));
    a.Np[l] = Np;
    for (int k0 = 0; k0 < Kp; k0 += KCH) {
      const int kc = std::min(KCH, Kp - k0);
      a.ch_layer[a.nch] = l;
      a.ch_k0[a.nch] = k0;
      a.ch_kc[a.nch] = kc;
      a.ch_off[a.nch] = (long long)off;
      off += (size_t)Np * kc * 2 * 2;
      ++a.nch;
    }
  }
  *total = off;
}

__global__ void k_pack_mlp(Args a, const float* __restrict__ theta, uint8_t* __restrict__ wpk) {
  const int q = blockIdx.y;
  const int l = a.ch_layer[q], k0 = a.ch_k0[q], kc = a.ch_kc[q], Np = a.Np[l];
  const int in = a.P.sizes[l], out = a.P.sizes[l + 1];
  __half* hi = reinterpret_cast<__half*>(wpk + a.ch_off[q]);
  __half* lo = hi + (size_t)Np * kc;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < Np * kc; idx += gridDim.x * blockDim.x) {
    const int r = idx / kc, k = idx % kc, kg = k0 + k;
    const float v = (r < out && kg < in) ? theta[a.P.w_off[l] + (size_t)r * in + kg] : 0.0f;
    const __half h = __float2half_rn(v);
    const __half e = __float2half_rn(v - __half2float(h));
    const int ci = tc::canon_idx(r, k, kc);
    hi[ci] = h;
    lo[ci] = e;
  }
}

// tanh(v) = sign(v) (1 - 2 / (e^{2|v|} + 1)): absolute error a few fp32 ulps of 1 everywhere (for
// tiny |v| that is a large relative error, but an activation enters the next layer's sums -- and
// the adjoint's 1 - h^2 -- through its absolute value, so the layer outputs keep fp32-class
// accuracy), ~7 instructions instead of tanhf's ~25.
__device__ __forceinline__ float tanh_fast(float v) {
  const float t = 1.0f - __fdividef(2.0f, __expf(2.0f * fabsf(v)) + 1.0f);
  return copysignf(t, v);
}

// hi/lo fp16 split of 2 consecutive K elements packed as one 32-bit TMEM word each
__device__ __forceinline__ void split_pair(float v0, float v1, uint32_t& hw, uint32_t& lw) {
  const __half2 h2 = __floats2half2_rn(v0, v1);
  const float2 hf = __half22float2(h2);
  const __half2 l2 = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
  hw = *reinterpret_cast<const uint32_t*>(&h2);
  lw = *reinterpret_cast<const uint32_t*>(&l2);
}

// Store a warp's 32 rows x 16 columns (row `lane` in v) to dst rows (row stride ld floats) with
// coalesced 64-byte row segments instead of one 16-byte piece per row per instruction: through a
// per-warp shared buffer, 8 rows per float4 store instruction.  rows_ok: rows of the warp that
// exist (< B).  dst + row * ld must be 16-byte aligned.
__device__ __forceinline__ void store_rows16(float* wb, const float* v, float* dst0, size_t ld, int rows_ok) {
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<float4*>(wb + lane * WB_LD + 4 * j) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int row = it * 8 + lane / 4, seg = lane % 4;
    if (row < rows_ok)
      *reinterpret_cast<float4*>(dst0 + (size_t)row * ld + 4 * seg) =
          *reinterpret_cast<const float4*>(wb + row * WB_LD + 4 * seg);
  }
  __syncwarp();
}

// The mirror image: load a warp's 32 rows x 16 columns (row `lane` into v) with coalesced 64-byte
// row segments; rows >= rows_ok read as 0.
__device__ __forceinline__ void load_rows16(float* wb, const float* src0, size_t ld, int rows_ok, float* v) {
  const int lane = threadIdx.x % 32;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int row = it * 8 + lane / 4, seg = lane % 4;
    const float4 x = row < rows_ok ? __ldg(reinterpret_cast<const float4*>(src0 + (size_t)row * ld + 4 * seg))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(wb + row * WB_LD + 4 * seg) = x;
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 x = *reinterpret_cast<const float4*>(wb + lane * WB_LD + 4 * j);
    v[4 * j] = x.x;
    v[4 * j + 1] = x.y;
    v[4 * j + 2] = x.z;
    v[4 * j + 3] = x.w;
  }
  __syncwarp();
}


__global__ void __launch_bounds__(THREADS, 1) k_mlp_fwd_tc(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NST], empty[NST], mma_done, a_ready;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float bias_s[BAGEL_MAX_LAYERS][BAGEL_MAX_WIDTH];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const PolicyDesc& P = a.P;
  const int L = P.n_layers;
  const int b0 = blockIdx.x * ROWS;
  if (warp == EPI_WARPS + 1) tc::tmem_alloc(&tmem_base, 512);
  for (int l = 0; l < P.n_layers; ++l)
    for (int o = tid; o < BAGEL_MAX_WIDTH; o += THREADS)
      bias_s[l][o] = o < P.sizes[l + 1] ? __ldg(a.theta + P.b_off[l] + o) : 0.0f;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&mma_done, 1);
    tc::mbar_init(&a_ready, 32 * EPI_WARPS);
    tc::fence_mbar_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == EPI_WARPS) {
    // ------------------------------------------------ weight producer (static operand: starts now)
    if (lane == 0) {
      for (int q = 0; q < a.nch; ++q) {
        const int s = q % NST;
        tc::mbar_wait(&empty[s], ((uint32_t)(q / NST) & 1u) ^ 1u);
        const uint32_t bytes = (uint32_t)a.Np[a.ch_layer[q]] * a.ch_kc[q] * 4u;
        tc::mbar_arrive_expect_tx(&full[s], bytes);
        tc::bulk_g2s(sm + (size_t)s * STAGE_BYTES, a.wpk + a.ch_off[q], bytes, &full[s]);
      }
    }
  } else if (warp == EPI_WARPS + 1) {
    // ------------------------------------------------ MMA issuer
    {  // the warp runs the loop; one elected lane issues each chunk's MMAs back to back
      int q = 0;
      for (int l = 0; l < L; ++l) {
        tc::mbar_wait(&a_ready, (uint32_t)l & 1u);  // this layer's input H is in TMEM
        tc::tc_fence_after();
        const uint32_t idesc = tc::idesc_f16(ROWS, a.Np[l]);
        bool first = true;
        for (; q < a.nch && a.ch_layer[q] == l; ++q) {
          const int s = q % NST, kc = a.ch_kc[q], k0 = a.ch_k0[q];
          tc::mbar_wait(&full[s], (uint32_t)(q / NST) & 1u);
          tc::tc_fence_after();
          const uint32_t base = tc::smem_u32(sm + (size_t)s * STAGE_BYTES);
          const uint32_t sbo = (uint32_t)(kc / 8) * 128u;
          const uint64_t bhi = tc::umma_desc(base, 128, sbo);
          const uint64_t blo = tc::umma_desc(base + (uint32_t)a.Np[l] * kc * 2u, 128, sbo);
          if (tc::elect_one()) {
            for (int ks = 0; ks < kc / 16; ++ks) {
              const uint64_t o = (uint64_t)(ks * 16);  // 256 bytes >> 4
              const uint32_t ac = (uint32_t)((k0 + 16 * ks) / 2);
              tc::mma_f16_ts(tmem + ACC, tmem + AHI + ac, bhi + o, idesc, (first && ks == 0) ? 0u : 1u);
              tc::mma_f16_ts(tmem + ACC, tmem + AHI + ac, blo + o, idesc, 1u);
              tc::mma_f16_ts(tmem + ACC, tmem + ALO + ac, bhi + o, idesc, 1u);
            }
            tc::umma_commit(&empty[s]);
          }
          __syncwarp();
          first = false;
        }
        if (tc::elect_one()) tc::umma_commit(&mma_done);
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue warps
    const int quarter = warp % 4, half = warp / 4;  // half: column group 0..3
    const int r = quarter * 32 + lane, b = b0 + r;
    const bool ok = b < a.B;
    const uint32_t tl = (uint32_t)(quarter * 32) << 16;
    float* act = ok ? a.act + (size_t)b * P.act_ld : nullptr;
    float* wb = reinterpret_cast<float*>(sm + NST * STAGE_BYTES) + warp * 32 * WB_LD;
    const int rows_ok = min(32, a.B - (b0 + quarter * 32));
    // layer-0 input phi = [x, g] or [x, g, g - x], zero-padded to 16 K elements
    if (half == 0) {
      const int n0 = P.sizes[0];
      float ph[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float v = 0.0f;
        if (ok && i < n0) {
          if (i < a.p) v = a.x[(size_t)b * a.p + i];
          else if (i < 2 * a.p) v = a.goals[(size_t)b * a.p + i - a.p];
          else v = a.goals[(size_t)b * a.p + i - 2 * a.p] - a.x[(size_t)b * a.p + i - 2 * a.p];
          act[P.aoff[0] + i] = v;
        }
        ph[i] = v;
      }
      uint32_t hw[8], lw[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) split_pair(ph[2 * e], ph[2 * e + 1], hw[e], lw[e]);
      tc::tmem_st8(tmem + tl + AHI, hw);
      tc::tmem_st8(tmem + tl + ALO, lw);
      tc::tmem_st_wait();
      if (ok)
        for (int c = 0; c < a.p; ++c) a.xstar[(size_t)b * a.D + c] = a.x[(size_t)b * a.p + c];
    }
    tc::tc_fence_before();
    tc::mbar_arrive(&a_ready);
    for (int l = 0; l < L; ++l) {
      const int out = P.sizes[l + 1], Np = a.Np[l];
      const bool last = l == L - 1;
      const float* bias = bias_s[l];
      tc::mbar_wait(&mma_done, (uint32_t)l & 1u);
      __syncwarp();
      tc::tc_fence_after();
      // this warp's columns: group `half` of 16-column chunks, chunk i going to group i % 4
      const int c_begin = 16 * half, c_step = 64, c_end = Np;
      for (int c0 = c_begin; c0 < c_end; c0 += c_step) {
        float v[16];
        tc::tmem_ld16(tmem + tl + ACC + (uint32_t)c0, v);
        tc::tmem_ld_wait();
        float bb[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // bias_s rows are zero-padded to 256 (16-byte loads, no bound checks)
          const float4 b4 = *reinterpret_cast<const float4*>(bias + c0 + 4 * j);
          bb[4 * j] = b4.x;
          bb[4 * j + 1] = b4.y;
          bb[4 * j + 2] = b4.z;
          bb[4 * j + 3] = b4.w;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = c0 + i < out ? tanh_fast(v[i] + bb[i]) : 0.0f;
        // activation tape: coalesced through the warp's staging buffer when aligned (warp-uniform)
        if (((P.act_ld | P.aoff[l + 1]) & 3) == 0 && c0 + 16 <= out) {
          store_rows16(wb, v, a.act + (size_t)(b0 + quarter * 32) * P.act_ld + P.aoff[l + 1] + c0, P.act_ld, rows_ok);
        } else if (ok) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < out) act[P.aoff[l + 1] + c0 + i] = v[i];
        }
        if (ok && last)
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c0 + i < out) a.xstar[(size_t)b * a.D + a.p + c0 + i] = v[i];
        if (!last) {
          uint32_t hw[8], lw[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) split_pair(v[2 * e], v[2 * e + 1], hw[e], lw[e]);
          tc::tmem_st8(tmem + tl + AHI + (uint32_t)(c0 / 2), hw);
          tc::tmem_st8(tmem + tl + ALO + (uint32_t)(c0 / 2), lw);
        }
      }
      if (!last) {
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&a_ready);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == EPI_WARPS + 1) tc::tmem_dealloc(tmem, 512);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_inval(&full[s]);
      tc::mbar_inval(&empty[s]);
    }
    tc::mbar_inval(&mma_done);
    tc::mbar_inval(&a_ready);
  }
}

// ---------------------------------------------------------------------------------------------
// The adjoint step of wide policies (a9) on the same machinery, per 128 rows:
//   xs-bar = sum_m xbar_m A_t[m];  dl_{L-1} = xs-bar[p:] (1 - u^2);
//   for l = L-1 .. 0:  hbar_l = dl_l W_l  (tcgen05: A = dl_l in TMEM, K = out_l; B = W_l^T rows,
//                      N = in_l);  l > 0: dl_{l-1} = hbar_l (1 - h_l^2) (tape + next A), else
//   xbar_t = carry xbar_{t+1} + xs-bar[:p] + dphi/dx^T hbar_0 + d(r_t / B)/dx_t.
// Backward chunks follow the forward ones in the packed buffer, layers in reverse order:
// B(r = i, k = o) = W_l[o][i], N = in_l rounded to 16 (>= 16), K = out_l rounded to 16.
struct BArgs {
  PolicyDesc P;
  RewardDesc rw;
  int p, D, B;
  const uint8_t* wpk;
  int nch;
  int ch_layer[MAXCH], ch_k0[MAXCH], ch_kc[MAXCH];
  long long ch_off[MAXCH];
  int Np[BAGEL_MAX_LAYERS];
  const float* goals;
  const float* x_t;     // B x p
  const float* A_t;     // B x p x D
  const float* act_t;   // B x act_ld
  float* delta_t;       // B x d_ld
  float* xbar;          // B x p (in: t + 1, out: t)
  float invB, carry;
};

void chunk_table_bwd(const PolicyDesc& P, BArgs& a, size_t base, size_t* total) {
  size_t off = base;
  a.nch = 0;
  for (int l = P.n_layers - 1; l >= 0; --l) {
    const int Kp = rup(P.sizes[l + 1], 16), Np = std::max(16, rup(P.sizes[l], 16));
    a.Np[l] = Np;
    for (int k0 = 0; k0 < Kp; k0 += KCH) {
      const int kc = std::min(KCH, Kp - k0);
      a.ch_layer[a.nch] = l;
      a.ch_k0[a.nch] = k0;
      a.ch_kc[a.nch] = kc;
      a.ch_off[a.nch] = (long long)off;
      off += (size_t)Np * kc * 2 * 2;
      ++a.nch;
    }
  }
  *total = off;
}

__global__ void k_pack_mlp_bwd(BArgs a, const float* __restrict__ theta, uint8_t* __restrict__ wpk) {
  const int q = blockIdx.y;
  const int l = a.ch_layer[q], k0 = a.ch_k0[q], kc = a.ch_kc[q], Np = a.Np[l];
  const int in = a.P.sizes[l], out = a.P.sizes[l + 1];
  __half* hi = reinterpret_cast<__half*>(wpk + a.ch_off[q]);
  __half* lo = hi + (size_t)Np * kc;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < Np * kc; idx += gridDim.x * blockDim.x) {
    const int r = idx / kc, k = idx % kc, kg = k0 + k;  // r = input unit i, kg = output unit o
    const float v = (r < in && kg < out) ? theta[a.P.w_off[l] + (size_t)kg * in + r] : 0.0f;
    const __half h = __float2half_rn(v);
    const __half e = __float2half_rn(v - __half2float(h));
    const int ci = tc::canon_idx(r, k, kc);
    hi[ci] = h;
    lo[ci] = e;
  }
}

__global__ void __launch_bounds__(THREADS, 1) k_mlp_bwd_tc(const __grid_constant__ BArgs a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NST], empty[NST], mma_done, a_ready;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const PolicyDesc& P = a.P;
  const int L = P.n_layers, p = a.p, D = a.D, q = P.sizes[L];
  const int b0 = blockIdx.x * ROWS;
  if (warp == EPI_WARPS + 1) tc::tmem_alloc(&tmem_base, 512);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&mma_done, 1);
    tc::mbar_init(&a_ready, 32 * EPI_WARPS);
    tc::fence_mbar_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == EPI_WARPS) {
    if (lane == 0) {
      for (int c = 0; c < a.nch; ++c) {
        const int s = c % NST;
        tc::mbar_wait(&empty[s], ((uint32_t)(c / NST) & 1u) ^ 1u);
        const uint32_t bytes = (uint32_t)a.Np[a.ch_layer[c]] * a.ch_kc[c] * 4u;
        tc::mbar_arrive_expect_tx(&full[s], bytes);
        tc::bulk_g2s(sm + (size_t)s * STAGE_BYTES, a.wpk + a.ch_off[c], bytes, &full[s]);
      }
    }
  } else if (warp == EPI_WARPS + 1) {
    {  // the warp runs the loop; one elected lane issues each chunk's MMAs back to back
      int c = 0;
      for (int j = 0; j < L; ++j) {
        const int l = L - 1 - j;
        tc::mbar_wait(&a_ready, (uint32_t)j & 1u);
        tc::tc_fence_after();
        const uint32_t idesc = tc::idesc_f16(ROWS, a.Np[l]);
        bool first = true;
        for (; c < a.nch && a.ch_layer[c] == l; ++c) {
          const int s = c % NST, kc = a.ch_kc[c], k0 = a.ch_k0[c];
          tc::mbar_wait(&full[s], (uint32_t)(c / NST) & 1u);
          tc::tc_fence_after();
          const uint32_t base = tc::smem_u32(sm + (size_t)s * STAGE_BYTES);
          const uint32_t sbo = (uint32_t)(kc / 8) * 128u;
          const uint64_t bhi = tc::umma_desc(base, 128, sbo);
          const uint64_t blo = tc::umma_desc(base + (uint32_t)a.Np[l] * kc * 2u, 128, sbo);
          if (tc::elect_one()) {
            for (int ks = 0; ks < kc / 16; ++ks) {
              const uint64_t o = (uint64_t)(ks * 16);  // 256 bytes >> 4
              const uint32_t ac = (uint32_t)((k0 + 16 * ks) / 2);
              tc::mma_f16_ts(tmem + ACC, tmem + AHI + ac, bhi + o, idesc, (first && ks == 0) ? 0u : 1u);
              tc::mma_f16_ts(tmem + ACC, tmem + AHI + ac, blo + o, idesc, 1u);
              tc::mma_f16_ts(tmem + ACC, tmem + ALO + ac, bhi + o, idesc, 1u);
            }
            tc::umma_commit(&empty[s]);
          }
          __syncwarp();
          first = false;
        }
        if (tc::elect_one()) tc::umma_commit(&mma_done);
        __syncwarp();
      }
    }
  } else {
    const int quarter = warp % 4, group = warp / 4;
    const int r = quarter * 32 + lane, b = b0 + r;
    const bool ok = b < a.B;
    const uint32_t tl = (uint32_t)(quarter * 32) << 16;
    float* wb = reinterpret_cast<float*>(sm + NST * STAGE_BYTES) + warp * 32 * WB_LD;
    const int rows_ok = min(32, a.B - (b0 + quarter * 32));
    // xs-bar_c = sum_m xbar_m A_t[m][c]
    float xs[BAGEL_MAX_D];
#pragma unroll
    for (int c = 0; c < BAGEL_MAX_D; ++c) {
      xs[c] = 0.0f;
      if (ok && c < D)
        for (int m = 0; m < p; ++m) xs[c] = fmaf(a.xbar[(size_t)b * p + m], a.A_t[((size_t)b * p + m) * D + c], xs[c]);
    }
    if (group == 0) {
      // dl_{L-1} = ubar (1 - u^2) (q <= 7 values, K padded to 16)
      float dv[16];
#pragma unroll
      for (int o = 0; o < 16; ++o) {
        float v = 0.0f;
#pragma unroll
        for (int c = 0; c < BAGEL_MAX_D; ++c)
          if (ok && o < q && c == p + o) {
            const float u = a.act_t[(size_t)b * P.act_ld + P.aoff[L] + o];
            v = xs[c] * (1.0f - u * u);
          }
        if (ok && o < q) a.delta_t[(size_t)b * P.d_ld + P.doff[L - 1] + o] = v;
        dv[o] = v;
      }
      uint32_t hw[8], lw[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) split_pair(dv[2 * e], dv[2 * e + 1], hw[e], lw[e]);
      tc::tmem_st8(tmem + tl + AHI, hw);
      tc::tmem_st8(tmem + tl + ALO, lw);
      tc::tmem_st_wait();
    }
    tc::tc_fence_before();
    tc::mbar_arrive(&a_ready);
    for (int j = 0; j < L; ++j) {
      const int l = L - 1 - j, in = P.sizes[l], Np = a.Np[l];
      tc::mbar_wait(&mma_done, (uint32_t)j & 1u);
      __syncwarp();
      tc::tc_fence_after();
      for (int c0 = 16 * group; c0 < Np; c0 += 64) {
        float v[16];
        tc::tmem_ld16(tmem + tl + ACC + (uint32_t)c0, v);
        tc::tmem_ld_wait();
        if (l > 0) {
          // dl_{l-1} = hbar (1 - h^2), h = layer l's input activations (tape)
          const bool vec = c0 + 16 <= in && ((P.act_ld | P.aoff[l] | P.d_ld | P.doff[l - 1]) & 3) == 0;
          if (vec) {  // warp-uniform: coalesced tape traffic through the warp's staging buffer
            float hv[16];
            load_rows16(wb, a.act_t + (size_t)(b0 + quarter * 32) * P.act_ld + P.aoff[l] + c0, P.act_ld, rows_ok, hv);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] *= 1.0f - hv[i] * hv[i];
            store_rows16(wb, v, a.delta_t + (size_t)(b0 + quarter * 32) * P.d_ld + P.doff[l - 1] + c0, P.d_ld, rows_ok);
          } else {
            const float* h = a.act_t + (size_t)b * P.act_ld + P.aoff[l] + c0;
            float* dst = a.delta_t + (size_t)b * P.d_ld + P.doff[l - 1] + c0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float hv = (ok && c0 + i < in) ? h[i] : 0.0f;
              v[i] = (c0 + i < in) ? v[i] * (1.0f - hv * hv) : 0.0f;
              if (ok && c0 + i < in) dst[i] = v[i];
            }
          }
          uint32_t hw[8], lw[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) split_pair(v[2 * e], v[2 * e + 1], hw[e], lw[e]);
          tc::tmem_st8(tmem + tl + AHI + (uint32_t)(c0 / 2), hw);
          tc::tmem_st8(tmem + tl + ALO + (uint32_t)(c0 / 2), lw);
        } else if (ok && c0 == 0) {
          // xbar_t = carry xbar_{t+1} + xs-bar[:p] + dphi/dx^T hbar_0 + d(r_t / B)/dx_t
          float qd = 0.0f;
          for (int c = 0; c < p; ++c) {
            const float df = a.x_t[(size_t)b * p + c] - a.goals[(size_t)b * p + c];
            qd = fmaf(a.rw.Q[c] * df, df, qd);
          }
          const float rr = expf(-qd * a.rw.inv_two_sr2);
          const float inv_sr2 = 2.0f * a.rw.inv_two_sr2;
#pragma unroll
          for (int c = 0; c < BAGEL_MAX_P; ++c) {
            if (c >= p) continue;
            float hb = 0.0f;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (i == c) hb += v[i];
              if (P.phi_mode == 1 && i == 2 * p + c) hb -= v[i];
            }
            float xsc = 0.0f;
#pragma unroll
            for (int cc = 0; cc < BAGEL_MAX_D; ++cc)
              if (cc == c) xsc = xs[cc];
            const float df = a.x_t[(size_t)b * p + c] - a.goals[(size_t)b * p + c];
            a.xbar[(size_t)b * p + c] = a.carry * a.xbar[(size_t)b * p + c] + xsc + hb + a.invB * rr * a.rw.Q[c] * df * inv_sr2;
          }
        }
      }
      if (l > 0) {
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&a_ready);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == EPI_WARPS + 1) tc::tmem_dealloc(tmem, 512);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_inval(&full[s]);
      tc::mbar_inval(&empty[s]);
    }
    tc::mbar_inval(&mma_done);
    tc::mbar_inval(&a_ready);
  }
}

size_t smem_bytes() { return NST * STAGE_BYTES + (size_t)EPI_WARPS * 32 * WB_LD * sizeof(float); }



}  // namespace mtc

bool mlp_tc_enabled(const bagel_ctx* c) {
  const char* env = getenv("BAGEL_MLP_TC");
  if (env && env[0] == '0') return false;
  int nch = 0;
  for (int l = 0; l < c->pol.n_layers; ++l) nch += (c->pol.sizes[l] + 15) / 16 * 16 / mtc::KCH + 1;
  return c->pol.sizes[0] <= 16 && nch <= mtc::MAXCH;
}

// Pack theta's weights into the chunked hi/lo operand (once per rollout; theta changes per iteration).
int mlp_tc_pack(bagel_ctx* c, const float* theta, cudaStream_t st) {
  mtc::Args a{};
  a.P = c->pol;
  size_t fwd = 0, total = 0;
  mtc::chunk_table(c->pol, a, &fwd);
  mtc::BArgs ab{};
  ab.P = c->pol;
  mtc::chunk_table_bwd(c->pol, ab, fwd, &total);
  if (c->ws.mlp_wpk_cap < total) {
    if (c->ws.mlp_wpk) cudaFree(c->ws.mlp_wpk);
    c->ws.mlp_wpk = nullptr;
    c->ws.mlp_wpk_cap = 0;
    if (cudaMalloc((void**)&c->ws.mlp_wpk, total) != cudaSuccess) return -1;
    c->ws.mlp_wpk_cap = total;
  }
  mtc::k_pack_mlp<<<dim3(16, a.nch), 256, 0, st>>>(a, theta, c->ws.mlp_wpk);
  mtc::k_pack_mlp_bwd<<<dim3(16, ab.nch), 256, 0, st>>>(ab, theta, c->ws.mlp_wpk);
  return 2;
}

// One adjoint step t of a wide policy on the tensor cores (replaces k_mlp_bwd; the caller runs
// k_xbar_init first and the steps t = T-1 .. 0).
int mlp_tc_backward_step(const bagel_ctx* c, const float* goals, int B, int t, long long B_global, cudaStream_t st) {
  static std::atomic<unsigned long long> devices{0};
  if (bagel_first_on_device(devices))
    cudaFuncSetAttribute(mtc::k_mlp_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mtc::smem_bytes());
  const Workspace& w = c->ws;
  mtc::Args af{};
  af.P = c->pol;
  size_t fwd = 0, total = 0;
  mtc::chunk_table(c->pol, af, &fwd);
  mtc::BArgs a{};
  a.P = c->pol;
  mtc::chunk_table_bwd(c->pol, a, fwd, &total);
  a.rw = c->rw;
  a.p = c->gp.p;
  a.D = c->gp.d;
  a.B = B;
  a.wpk = w.mlp_wpk;
  a.goals = goals;
  a.x_t = w.tape_x + (size_t)t * B * a.p;
  a.A_t = w.tape_A + (size_t)t * B * a.p * a.D;
  a.act_t = w.tape_act + (size_t)t * B * c->pol.act_ld;
  a.delta_t = w.tape_delta + (size_t)t * B * c->pol.d_ld;
  a.xbar = w.xbar;
  a.invB = (float)(1.0 / (double)B_global);
  a.carry = c->gp.abs_target ? 0.0f : 1.0f;
  mtc::k_mlp_bwd_tc<<<(B + mtc::ROWS - 1) / mtc::ROWS, mtc::THREADS, mtc::smem_bytes(), st>>>(a);
  return 1;
}

int mlp_tc_forward_step(const bagel_ctx* c, const float* theta, const float* goals, int B, int t, cudaStream_t st) {
  static std::atomic<unsigned long long> devices{0};
  if (bagel_first_on_device(devices))
    cudaFuncSetAttribute(mtc::k_mlp_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mtc::smem_bytes());
  const Workspace& w = c->ws;
  mtc::Args a{};
  a.P = c->pol;
  size_t total = 0;
  mtc::chunk_table(c->pol, a, &total);
  a.p = c->gp.p;
  a.D = c->gp.d;
  a.B = B;
  a.wpk = w.mlp_wpk;
  a.theta = theta;
  a.x = w.tape_x + (size_t)t * B * a.p;
  a.goals = goals;
  a.act = w.tape_act + (size_t)t * B * c->pol.act_ld;
  a.xstar = w.xstar;
  mtc::k_mlp_fwd_tc<<<(B + mtc::ROWS - 1) / mtc::ROWS, mtc::THREADS, mtc::smem_bytes(), st>>>(a);
  return 1;
}
