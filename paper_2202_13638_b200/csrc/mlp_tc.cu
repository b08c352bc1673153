// mlp_tc.cu -- the per-step policy forward (a1; tanh hidden and output, R13/R14)
// and its adjoint (a9) for WIDE policies (C3: 4-256-256-256-1) on the 5th-generation tensor cores.
//
// A cluster of CS = 4 CTAs owns 128 trajectories; every layer is split along its OUTPUT columns
// (16-column units, CTA `rank` computing units [u rank / CS, u (rank + 1) / CS)):
//   D[128 x out_slice] = H[128 x in] . W_l[out_slice]^T  on tcgen05 (kind::f16, fp32 TMEM
//   accumulator), with the same 3-pass fp16 split as the GP contraction (h = h_hi + h_lo, W = W_hi +
//   W_lo; h.W ~ h_hi W_hi + h_hi W_lo + h_lo W_hi, fp32-class accuracy, tests/test_gpu_tc.py);
//   A = H (hi | lo) in shared memory (canonical no-swizzle K-major, SS form), B = this CTA's rows of
//   the weight chunks, packed once per rollout (k_pack_mlp) and streamed by 1-D bulk copies
//   through a 3-stage ring.  The epilogue (bias + tanh, activation tape) splits its 128 x 64 slice
//   of the next layer's input into fp16 hi / lo, stores it locally as a contiguous region of the A
//   buffers, and one thread bulk-copies the region into the 3 peers (TMA engine, shared -> peer
//   shared, completing tx on the peer's per-region barrier), so the next layer's MMAs start on the
//   local region while the peers' regions arrive.  The MMA warps' completion is multicast to every
//   CTA's a_free barrier: nobody overwrites a region that a CTA's MMAs still read.
// 4x the CTAs of one-CTA-per-128-rows (C3: 128 instead of 32 SMs), a quarter of the weight bytes
// and of the MMA work per CTA.  Warps 0-15: epilogue (warp w: TMEM lane quarter w % 4, column
// group w / 4); warp 16: weight producer; warp 17: MMA issuer.
#include <cuda_fp16.h>
#include <stdlib.h>

#include <algorithm>

#include "bagel_internal.h"
#include "tc.cuh"

namespace mtc {

constexpr int ROWS = 128;
constexpr int CS = 4;            // CTAs per cluster (the column split of every layer)
constexpr int KCH = 64;          // K elements per pipeline stage
constexpr int NST = 3;           // ring stages (4 measured: no gain)
constexpr int EPI_WARPS = 16;    // 4 per TMEM lane quarter, each a 16-column group of the slice
constexpr int PROD_WARP = EPI_WARPS, MMA_WARP = EPI_WARPS + 1;
constexpr int THREADS = 32 * (EPI_WARPS + 2);
constexpr int MAXCH = 32;        // chunks over all layers (8 layers x 4 chunks of 64)
constexpr int SLICE = 64;        // columns per CTA at most: 256 / CS
constexpr size_t A_HALF = (size_t)ROWS * BAGEL_MAX_WIDTH * 2;           // one of hi / lo, fp16
constexpr size_t STAGE_BYTES = (size_t)SLICE * KCH * 2 * 2;            // hi + lo of 64 x 64 fp16
static_assert(BAGEL_MAX_WIDTH <= 16 * 4 * CS, "a CTA's slice must fit the 4 epilogue column groups");

// The output columns of a layer (Np of them, a multiple of 16) that CTA `rank` computes.
__host__ __device__ __forceinline__ void col_slice(int Np, int rank, int& cb, int& nl) {
  const int units = Np / 16, u0 = units * rank / CS, u1 = units * (rank + 1) / CS;
  cb = 16 * u0;
  nl = 16 * (u1 - u0);
}

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
  unsigned long long* dbg;       // optional event stamps of CTA 0 (bagel_debug_trace), else null
};

__device__ __forceinline__ void stamp(unsigned long long* d, int slot) {
  if (d && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    d[slot] = t;
  }
}

__host__ __device__ inline int rup(int a, int b) { return (a + b - 1) / b * b; }

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

// This thread's 16 consecutive values of one row (16-byte aligned) as 4 vector stores / loads.
__device__ __forceinline__ void store_row16(const float* v, float* dst) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
__device__ __forceinline__ void load_row16(const float* src, float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(src) + j);
    v[4 * j] = x.x;
    v[4 * j + 1] = x.y;
    v[4 * j + 2] = x.z;
    v[4 * j + 3] = x.w;
  }
}

// Hand this CTA's slice of the next layer's input to the cluster.  The A buffers hold that input
// as CS regions, region j = the columns [cb_j, cb_j + nl_j) computed by rank j, each a canonical
// K-major tile (KT = nl_j) at byte offset 256 cb_j of the hi / lo halves -- so a CTA's slice is
// contiguous.  Every epilogue thread stores its 16 values of row r locally; after a proxy fence and
// a barrier over the epilogue warps, one thread bulk-copies the region (TMA engine, smem -> peer
// smem) into every peer, completing tx on the peer's a_rdy[rank], and arms this CTA's own region
// barriers (a_rdy[j]: expect the peer's bytes; a_rdy[rank]: a plain arrive).
__device__ __forceinline__ void exchange_slice(uint8_t* Ahi, uint8_t* Alo, int rank, int Np, int r, int c0, bool have,
                                               const float* v, uint64_t* a_rdy) {
  int cb, nl;
  col_slice(Np, rank, cb, nl);
  if (have) {
    uint32_t hw[8], lw[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) split_pair(v[2 * e], v[2 * e + 1], hw[e], lw[e]);
    const size_t base = (size_t)256 * cb;
    const int o0 = 2 * tc::canon_idx(r, c0, nl), o1 = 2 * tc::canon_idx(r, c0 + 8, nl);
    *reinterpret_cast<uint4*>(Ahi + base + o0) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(Ahi + base + o1) = make_uint4(hw[4], hw[5], hw[6], hw[7]);
    *reinterpret_cast<uint4*>(Alo + base + o0) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    *reinterpret_cast<uint4*>(Alo + base + o1) = make_uint4(lw[4], lw[5], lw[6], lw[7]);
  }
  tc::fence_proxy_async();
  tc::named_sync(1, 32 * EPI_WARPS);
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(256 * nl);
    if (nl > 0)
      for (int d = 0; d < CS; ++d) {
        if (d == rank) continue;
        tc::bulk_s2s_cluster(Ahi + (size_t)256 * cb, Ahi + (size_t)256 * cb, bytes, &a_rdy[rank], (uint32_t)d);
        tc::bulk_s2s_cluster(Alo + (size_t)256 * cb, Alo + (size_t)256 * cb, bytes, &a_rdy[rank], (uint32_t)d);
      }
    for (int j = 0; j < CS; ++j) {
      int cbj, nlj;
      col_slice(Np, j, cbj, nlj);
      if (j == rank) tc::mbar_arrive(&a_rdy[j]);
      else tc::mbar_arrive_expect_tx(&a_rdy[j], (uint32_t)(2 * 256 * nlj));
    }
  }
}

// The same for this CTA's own A buffers only (the layer-0 input, built by every CTA).
__device__ __forceinline__ void put_a_row16_local(uint8_t* Ahi, uint8_t* Alo, int r, int k, int KT, const float* v) {
  uint32_t hw[8], lw[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) split_pair(v[2 * e], v[2 * e + 1], hw[e], lw[e]);
  const int o0 = 2 * tc::canon_idx(r, k, KT), o1 = 2 * tc::canon_idx(r, k + 8, KT);
  *reinterpret_cast<uint4*>(Ahi + o0) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  *reinterpret_cast<uint4*>(Ahi + o1) = make_uint4(hw[4], hw[5], hw[6], hw[7]);
  *reinterpret_cast<uint4*>(Alo + o0) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  *reinterpret_cast<uint4*>(Alo + o1) = make_uint4(lw[4], lw[5], lw[6], lw[7]);
}

// Weight producer (one lane): this CTA's rows of every chunk, hi and lo slices.
template <class A>
__device__ __forceinline__ void produce_weights(const A& a, int rank, uint8_t* ring, uint64_t* full, uint64_t* empty) {
  int i = 0;
  for (int q = 0; q < a.nch; ++q) {
    const int Np = a.Np[a.ch_layer[q]], kc = a.ch_kc[q];
    int cb, nl;
    col_slice(Np, rank, cb, nl);
    if (nl == 0) continue;
    const int s = i % NST;
    tc::mbar_wait(&empty[s], ((uint32_t)(i / NST) & 1u) ^ 1u);
    const uint32_t bytes = (uint32_t)nl * kc * 2u;
    tc::mbar_arrive_expect_tx(&full[s], 2u * bytes);
    uint8_t* dst = ring + (size_t)s * STAGE_BYTES;
    const uint8_t* src = a.wpk + a.ch_off[q] + (size_t)2 * cb * kc;
    tc::bulk_g2s(dst, src, bytes, &full[s]);
    tc::bulk_g2s(dst + bytes, src + (size_t)2 * Np * kc, bytes, &full[s]);
    ++i;
  }
}

// MMA issue for one layer (the warp runs it; one elected lane issues): D[128 x nl] = A[128 x K] B^T.
// Kin < 0: A is the locally built first-layer input (one canonical tile, KT = 16, ready on a0);
// else A is in CS regions (the slices of the previous layer's Kin = Np_prev outputs, see
// exchange_slice), region j waited on a_rdy[j] (parity ph) before its first K step, and every
// region's phase consumed before the function returns.
template <class A>
__device__ __forceinline__ void mma_layer(const A& a, int l, int Kin, int nl, int& q, int& i, uint32_t tmem,
                                          const uint8_t* Ahi, const uint8_t* Alo, uint8_t* ring, uint64_t* full,
                                          uint64_t* empty, uint64_t* a_rdy, uint32_t ph) {
  const uint32_t idesc = tc::idesc_f16(ROWS, nl > 0 ? nl : 16);
  const uint32_t ahi0 = tc::smem_u32(Ahi), alo0 = tc::smem_u32(Alo);
  uint32_t waited = 0;
  bool first = true;
  for (; q < a.nch && a.ch_layer[q] == l; ++q) {
    if (nl == 0) continue;
    const int s = i % NST, kc = a.ch_kc[q], k0 = a.ch_k0[q];
    tc::mbar_wait(&full[s], (uint32_t)(i / NST) & 1u);
    tc::tc_fence_after();
    const uint32_t base = tc::smem_u32(ring + (size_t)s * STAGE_BYTES);
    const uint32_t sbo = (uint32_t)(kc / 8) * 128u;
    const uint64_t bhi = tc::umma_desc(base, 128, sbo);
    const uint64_t blo = tc::umma_desc(base + (uint32_t)nl * kc * 2u, 128, sbo);
    if (tc::elect_one()) {
      for (int ks = 0; ks < kc / 16; ++ks) {
        const int k = k0 + 16 * ks;
        uint32_t aoff, asbo;
        if (Kin < 0) {
          aoff = (uint32_t)(k / 8) * 128u;
          asbo = 256u;
        } else {
          int j = 0, cbj = 0, nlj = 0;
          for (; j < CS; ++j) {
            col_slice(Kin, j, cbj, nlj);
            if (k < cbj + nlj) break;
          }
          if (!(waited & (1u << j))) {
            tc::mbar_wait(&a_rdy[j], ph);
            tc::tc_fence_after();
            waited |= 1u << j;
          }
          aoff = 256u * (uint32_t)cbj + (uint32_t)((k - cbj) / 8) * 128u;
          asbo = (uint32_t)(nlj / 8) * 128u;
        }
        const uint64_t ahi = tc::umma_desc(ahi0 + aoff, 128, asbo), alo = tc::umma_desc(alo0 + aoff, 128, asbo);
        const uint64_t o = (uint64_t)(ks * 16);  // 256 bytes >> 4 within the chunk
        tc::mma_f16(tmem, ahi, bhi + o, idesc, (first && ks == 0) ? 0u : 1u);
        tc::mma_f16(tmem, ahi, blo + o, idesc, 1u);
        tc::mma_f16(tmem, alo, bhi + o, idesc, 1u);
      }
      tc::umma_commit(&empty[s]);
    }
    __syncwarp();
    first = false;
    ++i;
  }
  // Consume every region's phase even where this CTA issued no MMA on it (nl = 0, or a region it
  // did not reach): a_free, committed after this, then certifies to the whole cluster that all
  // copies INTO this CTA have landed -- a CTA must not exit with a peer's copy still in flight.
  if (Kin >= 0)
    for (int j = 0; j < CS; ++j) tc::mbar_wait(&a_rdy[j], ph);
  tc::tc_fence_after();
}

__global__ void __launch_bounds__(THREADS, 1) k_mlp_fwd_tc(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[NST], empty[NST], mma_done, a_ready, a_free, a_rdy[CS];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float bias_s[BAGEL_MAX_LAYERS][BAGEL_MAX_WIDTH];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const PolicyDesc& P = a.P;
  const int L = P.n_layers;
  const int rank = (int)tc::cluster_rank();
  const int b0 = (blockIdx.x / CS) * ROWS;
  uint8_t* Ahi = sm;
  uint8_t* Alo = sm + A_HALF;
  uint8_t* ring = sm + 2 * A_HALF;
  if (tid == 0) stamp(a.dbg, 0);
  if (warp == MMA_WARP) tc::tmem_alloc(&tmem_base, SLICE);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&mma_done, 1);
    tc::mbar_init(&a_ready, EPI_WARPS);  // the locally built first layer's input
    tc::mbar_init(&a_free, CS);
    for (int j = 0; j < CS; ++j) tc::mbar_init(&a_rdy[j], 1);
    tc::fence_mbar_init();
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // every CTA's barriers exist before any remote arrive / store
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) stamp(a.dbg, 1);

  if (warp == PROD_WARP) {
    if (lane == 0) produce_weights(a, rank, ring, full, empty);
  } else if (warp == MMA_WARP) {
    int q = 0, i = 0;
    for (int l = 0; l < L; ++l) {
      int cb, nl;
      col_slice(a.Np[l], rank, cb, nl);
      if (l == 0) {
        tc::mbar_wait(&a_ready, 0u);
        tc::tc_fence_after();
      }
      if (lane == 0) stamp(a.dbg, 10 + 4 * l);
      mma_layer(a, l, l == 0 ? -1 : a.Np[l - 1], nl, q, i, tmem, Ahi, Alo, ring, full, empty, a_rdy,
                (uint32_t)(l - 1) & 1u);
      if (lane == 0) stamp(a.dbg, 11 + 4 * l);
      if (tc::elect_one()) {
        tc::umma_commit(&mma_done);
        tc::umma_commit_mc(&a_free, (uint16_t)((1u << CS) - 1u));
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ epilogue warps
    const int quarter = warp % 4, group = warp / 4;
    const int r = quarter * 32 + lane, b = b0 + r;
    const bool ok = b < a.B;
    const uint32_t tl = (uint32_t)(quarter * 32) << 16;
    float* act = ok ? a.act + (size_t)b * P.act_ld : nullptr;
    // layer-0 input phi = [x, g] or [x, g, g - x], zero-padded to 16 K elements (every CTA builds
    // its own copy; rank 0 writes the tape and x*)
    if (group == 0) {
      const int n0 = P.sizes[0];
      float ph[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float v = 0.0f;
        if (ok && i < n0) {
          if (i < a.p) v = a.x[(size_t)b * a.p + i];
          else if (i < 2 * a.p) v = a.goals[(size_t)b * a.p + i - a.p];
          else v = a.goals[(size_t)b * a.p + i - 2 * a.p] - a.x[(size_t)b * a.p + i - 2 * a.p];
          if (rank == 0) act[P.aoff[0] + i] = v;
        }
        ph[i] = v;
      }
      put_a_row16_local(Ahi, Alo, r, 0, 16, ph);
      tc::fence_proxy_async();
      if (ok && rank == 0)
        for (int c = 0; c < a.p; ++c) a.xstar[(size_t)b * a.D + c] = a.x[(size_t)b * a.p + c];
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&a_ready);
    // the biases (loaded while the first layer's MMAs run)
    for (int l = 0; l < P.n_layers; ++l)
      for (int o = tid; o < BAGEL_MAX_WIDTH; o += 32 * EPI_WARPS)
        bias_s[l][o] = o < P.sizes[l + 1] ? __ldg(a.theta + P.b_off[l] + o) : 0.0f;
    tc::named_sync(2, 32 * EPI_WARPS);
    for (int l = 0; l < L; ++l) {
      const int out = P.sizes[l + 1], Np = a.Np[l];
      const bool last = l == L - 1;
      int cb, nl;
      col_slice(Np, rank, cb, nl);
      const int c0 = 16 * group, col = cb + c0;  // this warp's 16 columns of the slice
      const bool have = c0 < nl;
      tc::mbar_wait(&mma_done, (uint32_t)l & 1u);
      __syncwarp();
      tc::tc_fence_after();
      if (warp == 0 && lane == 0) stamp(a.dbg, 40 + 4 * l);
      float v[16];
      if (have) {
        tc::tmem_ld16(tmem + tl + (uint32_t)c0, v);
        tc::tmem_ld_wait();
        const float* bias = bias_s[l];
        float bb[16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // bias_s rows are zero-padded to 256 (16-byte loads, no bound checks)
          const float4 b4 = *reinterpret_cast<const float4*>(bias + col + 4 * j);
          bb[4 * j] = b4.x;
          bb[4 * j + 1] = b4.y;
          bb[4 * j + 2] = b4.z;
          bb[4 * j + 3] = b4.w;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = col + i < out ? tanh_fast(v[i] + bb[i]) : 0.0f;
      }
      if (!last) {
        // the next layer's input first (its hand-off is on the critical path), the tapes after
        tc::tc_fence_before();
        tc::mbar_wait_cluster(&a_free, (uint32_t)l & 1u);  // every CTA's MMAs of layer l have read A
        if (warp == 0 && lane == 0) stamp(a.dbg, 41 + 4 * l);
        exchange_slice(Ahi, Alo, rank, Np, r, c0, have, v, a_rdy);
        if (warp == 0 && lane == 0) stamp(a.dbg, 42 + 4 * l);
      }
      if (have) {
        // activation tape: 16-byte row stores when aligned (warp-uniform)
        if (((P.act_ld | P.aoff[l + 1]) & 3) == 0 && col + 16 <= out) {
          if (ok) store_row16(v, act + P.aoff[l + 1] + col);
        } else if (ok) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (col + i < out) act[P.aoff[l + 1] + col + i] = v[i];
        }
        if (ok && last)
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (col + i < out) a.xstar[(size_t)b * a.D + a.p + col + i] = v[i];
      }
    }
  }
  // Exit only once every CTA's last-layer MMAs are done (a_free, multicast by each MMA warp): by
  // then all region copies this CTA sent have landed (the receivers' MMAs waited for them) and no
  // peer will address this CTA's shared memory again.
  if (warp < EPI_WARPS) tc::mbar_wait(&a_free, (uint32_t)(L - 1) & 1u);
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) stamp(a.dbg, 99);
  if (warp == MMA_WARP) tc::tmem_dealloc(tmem, SLICE);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_inval(&full[s]);
      tc::mbar_inval(&empty[s]);
    }
    tc::mbar_inval(&mma_done);
    tc::mbar_inval(&a_ready);
    tc::mbar_inval(&a_free);
    for (int j = 0; j < CS; ++j) tc::mbar_inval(&a_rdy[j]);
  }
}

// ---------------------------------------------------------------------------------------------
// The adjoint step of wide policies (a9) on the same machinery, per 128 rows:
//   xs-bar = sum_m xbar_m A_t[m];  dl_{L-1} = xs-bar[p:] (1 - u^2);
//   for l = L-1 .. 0:  hbar_l = dl_l W_l  (tcgen05: A = dl_l in shared memory, K = out_l; B = W_l^T rows,
//                      N = in_l, split over the cluster);  l > 0: dl_{l-1} = hbar_l (1 - h_l^2) (next A + tape), else
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
  __shared__ uint64_t full[NST], empty[NST], mma_done, a_ready, a_free, a_rdy[CS];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const PolicyDesc& P = a.P;
  const int L = P.n_layers, p = a.p, D = a.D, q = P.sizes[L];
  const int rank = (int)tc::cluster_rank();
  const int b0 = (blockIdx.x / CS) * ROWS;
  uint8_t* Ahi = sm;
  uint8_t* Alo = sm + A_HALF;
  uint8_t* ring = sm + 2 * A_HALF;
  if (warp == MMA_WARP) tc::tmem_alloc(&tmem_base, SLICE);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&mma_done, 1);
    tc::mbar_init(&a_ready, EPI_WARPS);  // the locally built first layer's input
    tc::mbar_init(&a_free, CS);
    for (int j = 0; j < CS; ++j) tc::mbar_init(&a_rdy[j], 1);
    tc::fence_mbar_init();
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == PROD_WARP) {
    if (lane == 0) produce_weights(a, rank, ring, full, empty);
  } else if (warp == MMA_WARP) {
    int c = 0, i = 0;
    for (int j = 0; j < L; ++j) {
      const int l = L - 1 - j;
      int cb, nl;
      col_slice(a.Np[l], rank, cb, nl);
      if (j == 0) {
        tc::mbar_wait(&a_ready, 0u);
        tc::tc_fence_after();
      }
      mma_layer(a, l, j == 0 ? -1 : a.Np[l + 1], nl, c, i, tmem, Ahi, Alo, ring, full, empty, a_rdy,
                (uint32_t)(j - 1) & 1u);
      if (tc::elect_one()) {
        tc::umma_commit(&mma_done);
        tc::umma_commit_mc(&a_free, (uint16_t)((1u << CS) - 1u));
      }
      __syncwarp();
    }
  } else {
    const int quarter = warp % 4, group = warp / 4;
    const int r = quarter * 32 + lane, b = b0 + r;
    const bool ok = b < a.B;
    const uint32_t tl = (uint32_t)(quarter * 32) << 16;
    // xs-bar_c = sum_m xbar_m A_t[m][c]  (every CTA, for its own use)
    float xs[BAGEL_MAX_D];
#pragma unroll
    for (int c = 0; c < BAGEL_MAX_D; ++c) {
      xs[c] = 0.0f;
      if (ok && c < D)
        for (int m = 0; m < p; ++m) xs[c] = fmaf(a.xbar[(size_t)b * p + m], a.A_t[((size_t)b * p + m) * D + c], xs[c]);
    }
    if (group == 0) {
      // dl_{L-1} = ubar (1 - u^2) (q <= 7 values, K padded to 16); rank 0 writes the tape
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
        if (ok && o < q && rank == 0) a.delta_t[(size_t)b * P.d_ld + P.doff[L - 1] + o] = v;
        dv[o] = v;
      }
      put_a_row16_local(Ahi, Alo, r, 0, 16, dv);
      tc::fence_proxy_async();
    }
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&a_ready);
    for (int j = 0; j < L; ++j) {
      const int l = L - 1 - j, in = P.sizes[l], Np = a.Np[l];
      int cb, nl;
      col_slice(Np, rank, cb, nl);
      const int c0 = 16 * group, col = cb + c0;
      const bool have = c0 < nl;
      const bool vec = l > 0 && col + 16 <= in && ((P.act_ld | P.aoff[l] | P.d_ld | P.doff[l - 1]) & 3) == 0;
      tc::mbar_wait(&mma_done, (uint32_t)j & 1u);
      __syncwarp();
      tc::tc_fence_after();
      float v[16];
      if (have) {
        tc::tmem_ld16(tmem + tl + (uint32_t)c0, v);
        tc::tmem_ld_wait();
        if (l > 0) {
          // dl_{l-1} = hbar (1 - h^2), h = layer l's input activations (tape); stored after the hand-off
          if (vec) {  // warp-uniform: 16-byte row loads
            float hv[16];
            if (ok) load_row16(a.act_t + (size_t)b * P.act_ld + P.aoff[l] + col, hv);
            else
#pragma unroll
              for (int i = 0; i < 16; ++i) hv[i] = 0.0f;
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] *= 1.0f - hv[i] * hv[i];
          } else {
            const float* h = a.act_t + (size_t)b * P.act_ld + P.aoff[l] + col;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float hv = (ok && col + i < in) ? h[i] : 0.0f;
              v[i] = (col + i < in) ? v[i] * (1.0f - hv * hv) : 0.0f;
            }
          }
        } else if (ok && col == 0) {
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
        tc::tc_fence_before();
        tc::mbar_wait_cluster(&a_free, (uint32_t)j & 1u);
        exchange_slice(Ahi, Alo, rank, Np, r, c0, have, v, a_rdy);
        if (have) {  // the adjoint tape dl_{l-1}
          if (vec) {
            if (ok) store_row16(v, a.delta_t + (size_t)b * P.d_ld + P.doff[l - 1] + col);
          } else if (ok) {
            float* dst = a.delta_t + (size_t)b * P.d_ld + P.doff[l - 1] + col;
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (col + i < in) dst[i] = v[i];
          }
        }
      }
    }
  }
  if (warp < EPI_WARPS) tc::mbar_wait(&a_free, (uint32_t)(L - 1) & 1u);  // see k_mlp_fwd_tc
  tc::tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) tc::tmem_dealloc(tmem, SLICE);
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_inval(&full[s]);
      tc::mbar_inval(&empty[s]);
    }
    tc::mbar_inval(&mma_done);
    tc::mbar_inval(&a_ready);
    tc::mbar_inval(&a_free);
    for (int j = 0; j < CS; ++j) tc::mbar_inval(&a_rdy[j]);
  }
}

size_t smem_bytes() { return 2 * A_HALF + NST * STAGE_BYTES; }

// cluster launch: CS CTAs per 128 rows
template <class K, class A>
static int launch_cl(K kern, const A& a, int B, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(((B + ROWS - 1) / ROWS) * CS), 1, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? 1 : -1;
}



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
  return mtc::launch_cl(mtc::k_mlp_bwd_tc, a, B, st);
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
  a.dbg = t == 10 && c->tcs.dbg2 ? c->tcs.dbg2 + 60000 : nullptr;  // clear of k_p2_tc's per-CTA stamps
  return mtc::launch_cl(mtc::k_mlp_fwd_tc, a, B, st);
}
