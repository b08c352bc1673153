// theta_tc.cu -- the parameter gradient of a wide policy on the tensor cores (SURVEY §8(a) a9:
// "theta-bar += sum delta h^T", "Compute grad_theta L via Autodiff").
//
// For every layer l, W-bar_l = sum_{k = (t, b)} delta_l[k] h_l[k]^T and b-bar_l = sum_k delta_l[k]: a
// dense contraction over the K = T B rows of the reverse pass's tapes (C3: K = 2,048,000 rows of
// 256-wide layers, 5.5e11 flops).  One CTA per (K block of TGT_RPB rows, job = layer x 128-output
// tile): 8 conversion warps read the fp32 tape rows (coalesced: consecutive outputs / inputs of one
// row), scale, split each value into fp16 hi + lo and scatter them, transposed, into the canonical
// K-major SS operands of the stage (A = delta^T: 128 outputs x 32 rows, B = h^T: in x 32 rows); one
// elected lane issues the 3-pass split MMAs (hi.hi + hi.lo + lo.hi, fp32 accumulate in TMEM,
// M = 128, N = in); the epilogue undoes the scales and writes the CTA's partial to theta_part
// [K block][n_params], summed over the K blocks in fixed order by k_reduce_grad (rollout.cu).
// Scales: each output's delta column is brought to max |delta| in [2^12, 2^13) by a power of two
// (a max pre-pass over the CTA's K block: delta ~ 1/B_global is far below fp16's normal range
// otherwise); tanh activations (|h| < 1) are scaled by 2^13, the layer-0 input phi by a power of
// two from its max.  The biases are summed by the conversion threads from the same unscaled fp32
// values.
// K blocks of 4,096 rows bound each TMEM chain at 768 MMA steps (the accumulator truncates,
// DESIGN.md R37: ~5e-5 relative).  The tape slices of 16 rows per stage arrive by 1-D bulk copies
// (TMA engine) into a raw fp32 ring; the per-column maxima come from one streaming pass over the
// adjoint tape (k_theta_colmax).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "bagel_internal.h"
#include "tc.cuh"

namespace tgt {

constexpr int KC = 16;           // tape rows per stage (one MMA K step)
constexpr int RST = 4;           // raw fp32 staging ring (bulk copies of the tape slices)
constexpr int OST = 4;           // converted operand ring (fp16 hi / lo, canonical K-major)
constexpr int CW = 8;            // conversion / epilogue warps
constexpr int MMA_WARP = CW, LOAD_WARP = CW + 1;
constexpr int THREADS = 32 * (CW + 2);
constexpr int RPB = 4096;        // tape rows per K block
constexpr int MAX_JOBS = 2 * BAGEL_MAX_LAYERS;
constexpr int MAXNP = 256;

struct Job {
  int layer, o0, out, in, np;  // outputs o0 .. o0 + 127 of `out`; in inputs padded to np (mult. of 16)
  int w_base, b_base;          // offsets of W_l and b_l in theta
  int doff, aoff;              // tape offsets of delta_l and h_l
  int dcopy, hcopy;            // floats per row bulk-copied: delta slice, h slice (multiples of 4)
};

// 2-D tensor maps (one per job and tape): box = KC rows x the job's delta / h slice, so each
// stage is ONE TMA copy per tape instead of one 1-D copy per row
struct Maps {
  CUtensorMap m[2 * MAX_JOBS];
};

struct Args {
  long long K;
  int n_params, act_ld, d_ld, phi_w;
  int njobs;
  Job jobs[MAX_JOBS];
  const float* act;
  const float* delta;
  const float* colmax;  // [K block][d_ld + 1]: max |delta| per tape column, then max |phi|
  float* part;          // [K block][n_params]
};

__device__ __forceinline__ float pow2_to(float amax, int target_exp, float* inv) {
  // 2^s such that amax 2^s lies in [2^(target_exp - 1), 2^target_exp); 1 for amax == 0
  if (!(amax > 0.0f)) {
    *inv = 1.0f;
    return 1.0f;
  }
  int e;
  frexpf(amax, &e);  // amax = f 2^e, f in [0.5, 1)
  *inv = ldexpf(1.0f, e - target_exp);
  return ldexpf(1.0f, target_exp - e);
}

// one 16-byte chunk (8 consecutive K elements of operand row r) of a canonical K-major tile of KC
__device__ __forceinline__ uint32_t chunk_off(int r, int kq) {
  return (uint32_t)((((r >> 3) * (KC / 8) + kq) << 6) + ((r & 7) << 3)) * 2u;
}

__device__ __forceinline__ void split8(const float* v, float sc, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float a = v[j] * sc, b = v[j + 1] * sc;
    const __half2 h2 = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h2);
    const __half2 l2 = __floats2half2_rn(a - hf.x, b - hf.y);
    h[j / 2] = *reinterpret_cast<const uint32_t*>(&h2);
    l[j / 2] = *reinterpret_cast<const uint32_t*>(&l2);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Per K block: max |delta| of every adjoint-tape column and max |phi| (the layer-0 input) -- the
// power-of-two operand scales of k_theta_grad_tc.  Streams whole tape rows (coalesced float4).
// float4 column groups of the adjoint tape a CTA covers: every layer's delta segment (<= 8 layers of
// <= 256 outputs, each padded to a multiple of 4) -- d_ld / 4 <= 520
constexpr int CM_U = (BAGEL_MAX_LAYERS * (BAGEL_MAX_WIDTH + 4) / 4 + 31) / 32;
__global__ void __launch_bounds__(256) k_theta_colmax(long long K, int d_ld, int act_ld, int phi_w,
                                                       const float* __restrict__ delta,
                                                       const float* __restrict__ act, float* __restrict__ colmax) {
  __shared__ float red[8][32 * CM_U];
  __shared__ float red_phi[8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long k0 = (long long)blockIdx.x * RPB, k1 = min(K, k0 + RPB);
  const int n4 = d_ld / 4;
  float mx[CM_U];
#pragma unroll
  for (int u = 0; u < CM_U; ++u) mx[u] = 0.0f;
  float pm = 0.0f;
  for (long long k = k0 + warp; k < k1; k += 8) {
    const float4* row = reinterpret_cast<const float4*>(delta + k * d_ld);
#pragma unroll
    for (int u = 0; u < CM_U; ++u) {
      const int c4 = lane + 32 * u;
      if (c4 < n4) {
        const float4 v = __ldg(row + c4);
        mx[u] = fmaxf(mx[u], fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
    }
    if (lane < phi_w) pm = fmaxf(pm, fabsf(__ldg(act + k * act_ld + lane)));
  }
  // per float4 column group (the scale of an output is the max over its group of 4 columns: a
  // power-of-two scale only needs an upper bound)
#pragma unroll
  for (int u = 0; u < CM_U; ++u)
    if (lane + 32 * u < n4) red[warp][lane + 32 * u] = mx[u];
  for (int o = 16; o > 0; o >>= 1) pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, o));
  if (lane == 0) red_phi[warp] = pm;
  __syncthreads();
  float* out = colmax + (size_t)blockIdx.x * (d_ld + 1);
  for (int c = threadIdx.x; c < d_ld; c += 256) {
    float m = 0.0f;
    for (int w = 0; w < 8; ++w) m = fmaxf(m, red[w][c / 4]);
    out[c] = m;
  }
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int w = 0; w < 8; ++w) m = fmaxf(m, red_phi[w]);
    out[d_ld] = m;
  }
}

__global__ void __launch_bounds__(THREADS, 1) k_theta_grad_tc(Args a, const __grid_constant__ Maps maps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t rfull[RST], rempty[RST], ofull[OST], oempty[OST], done;
  __shared__ uint32_t tmem_base;
  __shared__ float s_o[128], inv_o[128];
  __shared__ float bsum[KC / 8][128];
  const Job J = a.jobs[blockIdx.y];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const long long k0 = (long long)blockIdx.x * RPB, k1 = min(a.K, k0 + RPB);
  const int nst = (int)((k1 - k0 + KC - 1) / KC);
  const int rw = J.dcopy + J.hcopy;                  // floats per staged row [delta slice | h slice]
  const size_t raw_bytes = (size_t)KC * rw * 4;
  const size_t a_bytes = (size_t)128 * KC * 2;       // A hi (lo follows)
  const size_t b_bytes = (size_t)J.np * KC * 2;      // B hi (lo follows)
  const size_t op_bytes = 2 * a_bytes + 2 * b_bytes;
  uint8_t* raw = sm;                                 // RST x raw
  uint8_t* ops = sm + (size_t)RST * KC * (128 + MAXNP) * 4;  // OST x operands
  const int nout = min(128, J.out - J.o0);
  const float* colmax = a.colmax + (size_t)blockIdx.x * (a.d_ld + 1);
  float s_h, inv_h;
  {
    const float m = J.layer == 0 ? colmax[a.d_ld] : 1.0f;  // phi from the data, tanh otherwise
    s_h = pow2_to(m, 13, &inv_h);
  }

  if (tid == 0) {
    for (int s = 0; s < RST; ++s) {
      tc::mbar_init(&rfull[s], 1);
      tc::mbar_init(&rempty[s], 32 * CW);
    }
    for (int s = 0; s < OST; ++s) {
      tc::mbar_init(&ofull[s], 32 * CW);
      tc::mbar_init(&oempty[s], 1);
    }
    tc::mbar_init(&done, 1);
    tc::fence_mbar_init();
  }
  if (tid < 128) {
    float inv;
    s_o[tid] = pow2_to(tid < nout ? colmax[J.doff + J.o0 + tid] : 0.0f, 13, &inv);
    inv_o[tid] = inv;
  }
  if (warp == MMA_WARP) tc::tmem_alloc(&tmem_base, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tmem_base;

  if (warp == LOAD_WARP) {
    // ------------------------------------------------ raw staging: per row, the delta and h slices
    if (lane == 0) {
      for (int i = 0; i < nst; ++i) {
        const int s = i % RST;
        const long long r0 = k0 + (long long)i * KC;
        const int rows = (int)min((long long)KC, k1 - r0);
        tc::mbar_wait(&rempty[s], ((uint32_t)(i / RST) & 1u) ^ 1u);
        (void)rows;  // rows past K arrive zero-filled (and are counted) by the tensor copy
        tc::mbar_arrive_expect_tx(&rfull[s], (uint32_t)(KC * rw * 4));
        uint8_t* dst = raw + (size_t)s * raw_bytes;
        const uint32_t bar = tc::smem_u32(&rfull[s]);
        const int row = (int)r0;
        const CUtensorMap* md = &maps.m[2 * blockIdx.y];
        const CUtensorMap* mh = md + 1;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(md)), "r"(J.doff + J.o0), "r"(row), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(tc::smem_u32(dst + (size_t)KC * J.dcopy * 4)), "l"(reinterpret_cast<uint64_t>(mh)), "r"(J.aoff),
              "r"(row), "r"(bar)
            : "memory");
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------ MMA issue: the warp waits, one lane issues
    const uint32_t idesc = tc::idesc_f16(128, J.np);
    constexpr uint32_t SBO = (KC / 8) * 128;
    for (int i = 0; i < nst; ++i) {
      const int s = i % OST;
      tc::mbar_wait(&ofull[s], (uint32_t)(i / OST) & 1u);
      tc::tc_fence_after();
      const uint32_t base = tc::smem_u32(ops + (size_t)s * op_bytes);
      const uint64_t dahi = tc::umma_desc(base, 128, SBO), dalo = tc::umma_desc(base + (uint32_t)a_bytes, 128, SBO);
      const uint64_t dbhi = tc::umma_desc(base + (uint32_t)(2 * a_bytes), 128, SBO);
      const uint64_t dblo = tc::umma_desc(base + (uint32_t)(2 * a_bytes + b_bytes), 128, SBO);
      if (tc::elect_one()) {
        tc::mma_f16(tmem, dahi, dbhi, idesc, i > 0 ? 1u : 0u);
        tc::mma_f16(tmem, dahi, dblo, idesc, 1u);
        tc::mma_f16(tmem, dalo, dbhi, idesc, 1u);
        tc::umma_commit(&oempty[s]);
      }
      __syncwarp();
    }
    if (tc::elect_one()) tc::umma_commit(&done);
    __syncwarp();
  } else {
    // ------------------------------------------------ conversion: staged fp32 rows -> scaled fp16
    // hi/lo operands.  Items: A (o, kq) 128 x 2, then B (i, kq) np x 2; thread t: t, t + 256, ...
    const int nA = 128 * (KC / 8), nItems = nA + J.np * (KC / 8);
    static_assert(128 * (KC / 8) == 32 * CW, "thread t owns A item t (output t % 128, K chunk t / 128)");
    // the bias gradient sum_k delta[k][o] from the same unscaled fp32 values (thread t: output
    // t % 128, rows of K chunk t / 128 of every stage)
    float bacc = 0.0f;
    for (int i = 0; i < nst; ++i) {
      const int s = i % RST, so = i % OST;
      const int rows = (int)min((long long)KC, k1 - (k0 + (long long)i * KC));
      tc::mbar_wait(&rfull[s], (uint32_t)(i / RST) & 1u);
      tc::mbar_wait(&oempty[so], ((uint32_t)(i / OST) & 1u) ^ 1u);
      const float* src = reinterpret_cast<const float*>(raw + (size_t)s * raw_bytes);
      uint8_t* dst = ops + (size_t)so * op_bytes;
      for (int it = tid; it < nItems; it += 32 * CW) {
        const bool isA = it < nA;
        const int r = isA ? it % 128 : (it - nA) % J.np;
        const int kq = isA ? it / 128 : (it - nA) / J.np;
        const bool ok = isA ? r < nout : r < J.in;
        // staged stage = [delta box: KC rows x dcopy | h box: KC rows x hcopy]
        const float* col = isA ? src + r : src + KC * J.dcopy + r;
        const int ld = isA ? J.dcopy : J.hcopy;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rr = kq * 8 + j;
          v[j] = (ok && rr < rows) ? col[rr * ld] : 0.0f;
        }
        uint4 hi, lo;
        if (isA) {
#pragma unroll
          for (int j = 0; j < 8; ++j) bacc += v[j];
          split8(v, s_o[r], hi, lo);
          *reinterpret_cast<uint4*>(dst + chunk_off(r, kq)) = hi;
          *reinterpret_cast<uint4*>(dst + a_bytes + chunk_off(r, kq)) = lo;
        } else {
          split8(v, s_h, hi, lo);
          *reinterpret_cast<uint4*>(dst + 2 * a_bytes + chunk_off(r, kq)) = hi;
          *reinterpret_cast<uint4*>(dst + 2 * a_bytes + b_bytes + chunk_off(r, kq)) = lo;
        }
      }
      tc::fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
      __threadfence_block();    // the staged loads above have returned before the raw stage is released
      tc::mbar_arrive(&rempty[s]);
      tc::mbar_arrive(&ofull[so]);
    }
    // ---- biases: the K chunks of an output combined in chunk order
    bsum[tid / 128][tid % 128] = bacc;
    asm volatile("bar.sync 1, %0;" ::"n"(32 * CW) : "memory");
    if (tid < 128 && tid < nout) {
      float b = 0.0f;
      for (int q = 0; q < KC / 8; ++q) b += bsum[q][tid];
      a.part[(size_t)blockIdx.x * a.n_params + J.b_base + J.o0 + tid] = b;
    }
    // ---- epilogue: TMEM -> unscale -> this K block's partial of W_l rows o0 .. o0 + nout
    tc::mbar_wait(&done, 0);
    __syncwarp();
    tc::tc_fence_after();
    const int quarter = warp % 4, half = warp / 4;
    const int o = quarter * 32 + lane;
    const int cols = J.np / 2, c0 = half * cols;
    float* dstp = a.part + (size_t)blockIdx.x * a.n_params + J.w_base + (size_t)(J.o0 + o) * J.in;
    const float unscale = inv_o[o] * inv_h;
    for (int c = 0; c < cols; c += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(c0 + c)));
      tc::tmem_ld_wait();
      if (o < nout)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + c + u < J.in) dstp[c0 + c + u] = __uint_as_float(r[u]) * unscale;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) tc::tmem_dealloc(tmem, 256);
}

}  // namespace tgt

using namespace tgt;

// Wide policies (a layer of >= 128 outputs and inputs) take the tensor-core path.
bool theta_tc_enabled(const PolicyDesc& P) {
  for (int l = 0; l < P.n_layers; ++l)
    if (P.sizes[l + 1] >= 128 && P.sizes[l] >= 128) return true;
  return false;
}

int theta_tc_blocks(long long K) { return (int)std::max(1LL, (K + RPB - 1) / RPB); }
size_t theta_tc_colmax_floats(const PolicyDesc& P, long long K) { return (size_t)theta_tc_blocks(K) * (P.d_ld + 1); }

int theta_grad_tc(const PolicyDesc& P, long long K, const float* act, const float* delta, float* colmax,
                  float* part, cudaStream_t st) {
  static std::atomic<unsigned long long> devices{0};
  const size_t smem = (size_t)RST * KC * (128 + MAXNP) * 4 + (size_t)OST * (2 * 128 * KC * 2 + 2 * MAXNP * KC * 2);
  if (bagel_first_on_device(devices)) bagel_set_smem_attr(k_theta_grad_tc, smem);
  Args a{};
  a.K = K;
  a.n_params = P.n_params;
  a.act_ld = P.act_ld;
  a.d_ld = P.d_ld;
  a.phi_w = P.sizes[0];
  a.act = act;
  a.delta = delta;
  a.colmax = colmax;
  a.part = part;
  int nj = 0, off = 0;
  for (int l = 0; l < P.n_layers; ++l) {
    const int in = P.sizes[l], out = P.sizes[l + 1];
    for (int o0 = 0; o0 < out; o0 += 128) {
      Job& j = a.jobs[nj++];
      j.layer = l;
      j.o0 = o0;
      j.out = out;
      j.in = in;
      j.np = (in + 15) / 16 * 16;
      j.w_base = off;
      j.b_base = off + in * out;
      j.doff = P.doff[l];
      j.aoff = P.aoff[l];
      j.dcopy = (std::min(128, out - o0) + 3) / 4 * 4;  // 16-byte multiples (tape segments are padded)
      j.hcopy = (in + 3) / 4 * 4;
    }
    off += in * out + out;
  }
  a.njobs = nj;
  const int nblk = theta_tc_blocks(K);
  k_theta_colmax<<<nblk, 256, 0, st>>>(K, P.d_ld, P.act_ld, P.sizes[0], delta, act, colmax);
  const dim3 grid(nblk, nj);
  // tensor maps: the adjoint / activation tapes as 2-D (columns, rows) fp32 arrays
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {  // thread-safe one-time lookup
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&f), cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return f;
  }();
  if (!encode) return -1;
  Maps maps;  // per call (no shared host state between contexts)
  for (int j = 0; j < nj; ++j) {
    for (int t = 0; t < 2; ++t) {
      const bool isd = t == 0;
      const cuuint64_t ld = (cuuint64_t)(isd ? P.d_ld : P.act_ld);
      const cuuint64_t dims[2] = {ld, (cuuint64_t)K};
      const cuuint64_t strides[1] = {ld * 4};
      const cuuint32_t box[2] = {(cuuint32_t)(isd ? a.jobs[j].dcopy : a.jobs[j].hcopy), (cuuint32_t)KC};
      const cuuint32_t es[2] = {1, 1};
      if (encode(&maps.m[2 * j + t], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(isd ? delta : act), dims,
                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -1;
    }
  }
  k_theta_grad_tc<<<grid, THREADS, smem, st>>>(a, maps);
  return 2;
}
