// gp_step_tc.cu -- the GP step of the rollout on the 5th-generation tensor cores
// (north star item (2): "a fused sm_100a kernel that generates k(x*,X) tiles on the
// fly in shared memory ... and contracts them against [alpha | R^T] staged by TMA on
// tensor cores ... it also emits the input Jacobians").
//
// Per output m and a batch of query rows x* (Eq.2-3 with LOVE):
//   pass 1 (k_p1_tc)  z = R k(x*, X) on tcgen05 (3-pass fp16 hi/lo split, fp32 TMEM
//                     accumulation); the 1 + d mean columns [mu | sum k a (x*_c - X_c)] are
//                     accumulated in fp32 on the CUDA cores by the same warps that
//                     generate ktilde = exp2(-||x_hat - X_hat||^2) (never stored in HBM).
//   reduce 1          sums the N-split partials; v = s - ||z||^2, sigma, J^mu; packs
//                     z as the fp16 hi/lo A operand of pass 2.
//   pass 2 (k_p2_tc)  W = Z R (w_n = sum_j z_j R_jn) on tcgen05, then on the CUDA cores
//                     sum_n w_n k_n [1 | X_n] for J^v (ktilde regenerated).
// Operands are packed once at cache-build time in the canonical no-swizzle K-major
// layout (tc.cuh) so every pipeline stage is ONE contiguous 1-D bulk copy (TMA engine).
// Split precision: a = hi + lo with hi = fp16(a), lo = fp16(a - hi); the product
// a.b ~ hi.hi + hi.lo + lo.hi (fp32 accumulate) -- fp32-class accuracy (SURVEY §7
// hard part 1), verified in tests/test_gpu_tc.py.  B operands carry power-of-two
// scales (per z column in pass 1, per training point in pass 2; per row for Z),
// undone exactly in the epilogues.
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "bagel_internal.h"
#include "policy_rows.cuh"
#include "tc.cuh"

namespace tcg {

constexpr int KT1 = 32;      // training points per pass-1 stage
constexpr int ST1 = 6;       // pass-1 ring stages (max): A (ktilde) and B (R tile halves), shared memory

constexpr int AUXW = 20;     // floats of per-n side data per stage row
constexpr int NT2 = 128;     // training points per pass-2 tile (the MMA N dimension)
constexpr int KS2 = 64;      // j per pass-2 K slab (one pipeline stage)
constexpr int ST2 = 8;       // pass-2 slab ring stages (Z lives in TMEM; each CTA of a pair holds half a slab)
constexpr int STX2 = 2;      // pass-2 aux ring stages (one per tile)
constexpr int STA = 8;       // pass-1 aux (per-n side data) ring stages
constexpr int P1_MAX_TILES = 80;  // longest pass-1 accumulation chain (N-tiles of KT1 points per split; C3 keeps S1 = 2)
constexpr int CTRL_WARPS = 3; // B producer, MMA issuer, aux producer
constexpr int GEN_WARPS = 16; // generator / epilogue warps (4 per TMEM lane quarter)
constexpr int THREADS = 32 * CTRL_WARPS + 32 * GEN_WARPS;
constexpr int P2_LD = 1 + BAGEL_MAX_D;

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }
__host__ __device__ inline int cdiv_dev(int a, int b) { return (a + b - 1) / b; }
// pass-1 ring depth for NC z-column tiles per CTA pair (NC = 1: A in TMEM, stage = B halves 16 KB;
// NC = 2: stage = A 16 KB + 2 x 16 KB of B halves in shared memory)
__host__ __device__ constexpr int p1_stages(int NC) { return NC > 1 ? 4 : 6; }
constexpr int A1C = 32;      // TMEM columns of one A stage when A lives in TMEM (NC = 1): hi (16) | lo (16)

struct Geo {
  int N, d, p, k;
  int nct, NZ;        // pass-1 z-column tiles and their width (<= 256, multiple of 16)
  int njt, KJ;        // pass-2 j tiles (<= 256, multiple of KS2)
  int nt1, nt2;       // number of n-tiles of pass 1 / pass 2
  size_t t1_bytes;    // bytes of one pass-1 stage tile [B hi | B lo | aux]
  size_t t2_bytes;    // bytes of one pass-2 stage tile
};

__host__ __device__ inline size_t t1_bytes(int NZ) { return (size_t)4 * NZ * KT1 + (size_t)KT1 * AUXW * 4; }
__host__ __device__ inline size_t t2_bytes(int KJ) { return (size_t)4 * NT2 * KJ + (size_t)NT2 * AUXW * 4; }

inline Geo make_geo(int N, int d, int p, int k) {
  Geo g{};
  g.N = N; g.d = d; g.p = p; g.k = k;
  g.nct = cdiv(k, 256);
  g.NZ = cdiv(cdiv(k, g.nct), 32) * 32;  // CTA pairs: each CTA holds NZ/2 columns of B
  g.njt = cdiv(k, 256);
  g.KJ = cdiv(cdiv(k, g.njt), KS2) * KS2;
  g.nt1 = cdiv(N, KT1);
  g.nt2 = cdiv(N, NT2);
  g.t1_bytes = t1_bytes(g.NZ);
  g.t2_bytes = t2_bytes(g.KJ);
  return g;
}

// Per-training-point side data ("aux") of a stage tile, pair-interleaved: points 2j and 2j + 1
// share a block of 2 x AUXW floats, field-major, point-minor -- so one float4 holds two fields
// of both points, i.e. the two lanes of two fp32x2 operands.
__host__ __device__ inline int aux_idx(int nn, int f) { return ((nn >> 1) * AUXW + f) * 2 + (nn & 1); }

// Every split operand is carried at 2^14 times its (power-of-two normalised) value: fp16's normal
// range starts at 2^-14, so the lo half of a value x (|lo| ~ 2^-12 |x|) stays normal -- i.e. keeps
// its 11 significant bits -- down to |x| ~ 2^-16 instead of 2^-2 of the operand's scale.  Without
// it, every ktilde < 1/4 (most of the training points a query sees) and every small R / z entry lost
// precision to the absolute 2^-25 spacing of fp16 subnormals.  Values stay below 2^14 < 65504.
// The 2^14 factors are exact and are undone in the epilogues (colscale, zrow_inv, aux 2^f_n).
constexpr float SPLIT_UP = 16384.0f, SPLIT_DOWN = 1.0f / 16384.0f;

__device__ __forceinline__ void split_f16(float v, __half& hi, __half& lo) {
  hi = __float2half_rn(v);
  lo = __float2half_rn(v - __half2float(hi));
}

// power-of-two scale bringing max|v| into [0.5, 1): returns 2^-e (and the inverse 2^e)
__device__ __forceinline__ float pow2_scale_for(float amax, float* inv) {
  if (!(amax > 0.0f)) {
    *inv = 1.0f;
    return 1.0f;
  }
  int e;
  frexpf(amax, &e);  // amax = f 2^e, f in [0.5, 1)
  *inv = ldexpf(1.0f, e);
  return ldexpf(1.0f, -e);
}

// ====================================================================== packing
// Pass-1 tiles of output m: [ct][t] -> [B hi: NZ x KT1 | B lo | aux: KT1 x AUXW]
// B(j, n) = s R_jn * colscale_j^-1 (j = ct*NZ + row), aux(n) = [X(d) | s alpha] (rest of the row 0).
__global__ void k_pack1(Geo g, const float* __restrict__ X, const double* __restrict__ alpha,
                        const double* __restrict__ R, double s, const float* __restrict__ qscale,
                        const float* __restrict__ colscale_inv, uint8_t* __restrict__ out) {
  const int t = blockIdx.x, ct = blockIdx.y;
  uint8_t* tile = out + ((size_t)ct * g.nt1 + t) * g.t1_bytes;
  __half* bhi = reinterpret_cast<__half*>(tile);
  __half* blo = bhi + (size_t)g.NZ * KT1;
  float* aux = reinterpret_cast<float*>(blo + (size_t)g.NZ * KT1);
  for (int idx = threadIdx.x; idx < g.NZ * KT1; idx += blockDim.x) {
    const int jr = idx / KT1, nn = idx % KT1;
    const int j = ct * g.NZ + jr, n = t * KT1 + nn;
    float v = 0.0f;
    if (j < g.k && n < g.N) v = (float)(s * R[(size_t)j * g.N + n]) * colscale_inv[j];
    __half hi, lo;
    split_f16(v, hi, lo);
    const int ci = tc::canon_idx(jr, nn, KT1);
    bhi[ci] = hi;
    blo[ci] = lo;
  }
  for (int idx = threadIdx.x; idx < KT1 * AUXW; idx += blockDim.x) {
    const int nn = idx / AUXW, f = idx % AUXW;
    const int n = t * KT1 + nn;
    float v = 0.0f;
    if (n < g.N) {
      if (f < g.d) v = X[(size_t)n * g.d + f];  // raw X: the exponent differences before scaling
      else if (f == g.d) v = (float)(s * alpha[n]);
    } else if (f < g.d) {
      v = 1e18f;  // padded training point: infinitely far, ktilde = 0
    }
    aux[aux_idx(nn, f)] = v;
  }
}

// Per-column (j) power-of-two scales of s R_j (max over n): colscale_inv = 2^-e_j, colscale = 2^e_j.
__global__ void k_colscale(const double* __restrict__ R, int N, int k, double s, float* __restrict__ cs_inv,
                           float* __restrict__ cs) {
  const int j = blockIdx.x;
  __shared__ float red[256];
  float a = 0.0f;
  for (int n = threadIdx.x; n < N; n += 256) a = fmaxf(a, fabsf((float)(s * R[(size_t)j * N + n])));
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    float inv;
    const float sc = pow2_scale_for(red[0], &inv);
    cs_inv[j] = sc * SPLIT_UP;                // B operand at 2^14 x its normalised value
    cs[j] = inv * (SPLIT_DOWN * SPLIT_DOWN);  // undoes the column scale and both operands' 2^14
  }
}

// Pass-2 tiles of output m: [jt][t] -> KJ/KS2 slabs [B hi: NT2 x KS2 | B lo: NT2 x KS2] (canonical
// K-major, rows = training points, K = j), then aux: NT2 x AUXW.
// B(n, j) = s R_jn * 2^-f_n (f_n from max over the tile's j range), aux(n) = [X(d) | 2^f_n].
__global__ void k_pack2(Geo g, const float* __restrict__ X, const double* __restrict__ R, double s,
                        const float* __restrict__ qscale, uint8_t* __restrict__ out) {
  const int t = blockIdx.x, jt = blockIdx.y;
  uint8_t* tile = out + ((size_t)jt * g.nt2 + t) * g.t2_bytes;
  __half* slabs = reinterpret_cast<__half*>(tile);
  float* aux = reinterpret_cast<float*>(tile + (size_t)4 * NT2 * g.KJ);
  __shared__ float rsc[NT2], rinv[NT2];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int nn = warp; nn < NT2; nn += blockDim.x / 32) {
    const int n = t * NT2 + nn;
    float a = 0.0f;
    if (n < g.N)
      for (int jr = lane; jr < g.KJ; jr += 32) {
        const int j = jt * g.KJ + jr;
        if (j < g.k) a = fmaxf(a, fabsf((float)(s * R[(size_t)j * g.N + n])));
      }
    for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0) {
      float inv;
      rsc[nn] = pow2_scale_for(a, &inv) * SPLIT_UP;
      rinv[nn] = inv * SPLIT_DOWN;
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < NT2 * g.KJ; idx += blockDim.x) {
    const int jr = idx / NT2, nn = idx % NT2;  // coalesced reads of R rows
    const int n = t * NT2 + nn, j = jt * g.KJ + jr;
    float v = 0.0f;
    if (n < g.N && j < g.k) v = (float)(s * R[(size_t)j * g.N + n]) * rsc[nn];
    __half hi, lo;
    split_f16(v, hi, lo);
    const int sl = jr / KS2, jj = jr % KS2;
    __half* sb = slabs + (size_t)sl * 2 * NT2 * KS2;
    const int ci = tc::canon_idx(nn, jj, KS2);
    sb[ci] = hi;
    sb[NT2 * KS2 + ci] = lo;
  }
  for (int idx = threadIdx.x; idx < NT2 * AUXW; idx += blockDim.x) {
    const int nn = idx / AUXW, f = idx % AUXW;
    const int n = t * NT2 + nn;
    float v = 0.0f;
    if (n < g.N) {
      if (f < g.d) v = X[(size_t)n * g.d + f];
      else if (f == g.d) v = rinv[nn];
    } else if (f < g.d) {
      v = 1e18f;
    }
    aux[aux_idx(nn, f)] = v;
  }
}

// ====================================================================== pass 1
struct P1Args {
  Geo g;
  int m_count;               // p
  const float* xstar;        // B x d
  int B;
  const uint8_t* tiles;      // [m][ct][t] pass-1 tiles
  size_t m_stride;           // bytes per output m of tiles
  int tiles_per_split;
  float* P1z;                // [split][m][ct][NZ][B]
  float* P1h;                // [split][m][B][1 + d]
  float qscale[BAGEL_MAX_P][BAGEL_MAX_D];
  unsigned long long* dbg;   // nullable: per-CTA %globaltimer event stamps (16 per CTA)
  // fused reduce 1 (cluster of the S1 splits, nct == 1): the outputs of k_r1a_tc + k_r1b_tc
  const float* colscale;     // [m][k] 2^e_j
  float s[BAGEL_MAX_P];
  float ell2inv[BAGEL_MAX_P][BAGEL_MAX_D];
  uint8_t* Zp;
  float* zrow_inv;
  float* mu;
  float* var;
  float* jmu;                // nullable
  float* sig;                // nullable
  unsigned long long* gbar;  // grid barrier counter
  int* err_flag;             // barrier watchdog report
  int diag;                  // timing experiments only (results invalid): 1 skip generator math, 2 skip MMAs
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp(unsigned long long* dbg, int k) {
  if (dbg) {
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    dbg[cta * 16 + k] = gtimer();
  }
}

// Grid-wide barrier of a one-wave grid (every CTA resident: grid <= #SM x occupancy, checked on
// the host; with programmatic dependent launch the next kernel's CTAs are only admitted after
// every CTA of this one has started).  One release-add per CTA on a counter that only grows
// (each launch adds G; zeroed whenever the grid shape changes), then an acquire-poll until the
// count reaches the next multiple of G.  The release (cumulative over the CTA's writes ordered
// before it by bar.sync) and the acquire make every CTA's writes before the barrier visible to
// every CTA after it.  Watchdog: if the grid is not co-resident after all (another context or
// stream holding SMs), the poll gives up after ~2 s and reports BAGEL_BARRIER_TIMEOUT through
// err_flag instead of hanging the device.
constexpr int GB_STRIDE = 32;   // unsigned long longs reserved per counter set
// Split phase: grid_arrive (after a __syncthreads: this CTA's writes are released) returns the
// target thread 0 must see; work that does not depend on other CTAs can run between the two.
__device__ __forceinline__ unsigned long long grid_arrive(unsigned long long* ctr) {
  __syncthreads();
  unsigned long long target = 0;
  if (threadIdx.x == 0) {
    const unsigned long long G = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
    target = (old / G + 1) * G;
  }
  return target;
}
__device__ __forceinline__ void grid_wait(unsigned long long* ctr, unsigned long long target, int* err_flag) {
  if (threadIdx.x == 0) {
    unsigned long long cur, t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(ctr) : "memory");
      if (cur >= target) break;
      if ((++spins & 1023u) == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > 2000000000ull) {
          if (err_flag) atomicMin(err_flag, BAGEL_BARRIER_TIMEOUT);
          break;
        }
      }
    } while (true);
  }
  __syncthreads();
}
__device__ __forceinline__ void grid_barrier(unsigned long long* ctr, int* err_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long G = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
    const unsigned long long target = (old / G + 1) * G;
    unsigned long long cur, t0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    unsigned spins = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(ctr) : "memory");
      if (cur >= target) break;
      if ((++spins & 1023u) == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > 2000000000ull) {
          if (err_flag) atomicMin(err_flag, BAGEL_BARRIER_TIMEOUT);
          break;
        }
      }
    } while (true);
  }
  __syncthreads();
}

// Packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2 on sm_100a): two independent lanes, each
// rounded exactly as the scalar instruction would.
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// Programmatic dependent launch: let the next kernel of the stream be scheduled now (its CTAs
// land as SMs free up), and wait for the previous kernel's completion and memory flush before
// touching anything it wrote.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// fields 0 .. NV-1 of training points 2j, 2j + 1 (pair block at `pair`) as float2 lanes
template <int NV>
__device__ __forceinline__ void load_aux2(const float* pair, float2* out) {
#pragma unroll
  for (int v = 0; v < (NV + 1) / 2; ++v) {
    const float4 f = *reinterpret_cast<const float4*>(pair + 4 * v);
    out[2 * v] = make_float2(f.x, f.y);
    if (2 * v + 1 < NV) out[2 * v + 1] = make_float2(f.z, f.w);
  }
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// FUSED (nct == 1, cooperative launch: every CTA is resident): after the MMAs each CTA parks its
// partial z tile in its idle stage memory, writes it row-major to P1z (coalesced), and after a
// grid-wide barrier every warp reduces whole rows over the S1 partials in split order and
// finishes them as reduce 1 does (v, sigma, J^mu, row scale, packed Z): the two reduce launches
// (and their column-strided passes over the partials) disappear.  (A DSMEM cluster reduction was
// measured first: cluster residency caps S1 at 6 here and DSMEM moves ~20 B/clk/SM -- slower.)
template <int D>
struct P1Shared {
  uint64_t full_a[ST1], full_b[ST1], pfull_b[ST1], empty[ST1], full_x[STA], empty_x[STA], done;
  float hsum[3][128][1 + D];
};

// Pass 1 of the CTA with grid coordinates (bx, by, bz) on CTA pairs (cta_group::2): the two CTAs
// of a cluster along x (row tiles 2c, 2c + 1) share (output m, column-tile pair ctp, split) and run
// ONE chain of M = 256 MMAs issued by the leader (rank 0), SS form.  Each CTA's generator warps
// write the ktilde hi/lo A operand of ITS 128 rows to its own shared memory (canonical K-major,
// st.shared + proxy fence); each CTA holds HALF of the z columns of every R tile (B); the pair
// computes NC = min(2, nct - 2 ctp) column tiles of NZ columns at once (accumulators NC x NZ TMEM
// columns in each CTA), so at k = 512 (C4, C5) every ktilde is generated once per row instead of
// once per column tile, and the MMA runs at the pair floor (profiles/r02_b_tc_pair_issue_rate.txt).
// FUSED: the partial z tile is parked in shared memory and the rows this CTA does not finish are
// written to P1z (p1_reduce runs after a grid barrier).  Ends with every thread past a
// __syncthreads and the barriers retired.
template <int D, bool FUSED>
__device__ __forceinline__ void p1_main(const P1Args& a, const int bx, const int by, const int bz, const int nbz,
                                        uint8_t* sm, P1Shared<D>& sh, const uint32_t tmem) {
  const Geo& g = a.g;
  const int NZ = g.NZ;
  constexpr int NAUX = D + 1;  // X_n (d) | s alpha_n
  const int nctp = cdiv_dev(g.nct, 2);
  const int m = by / nctp, ctp = by % nctp, ct0 = 2 * ctp;
  const int NC = min(2, g.nct - ct0);
  // NC = 1 (k <= 256, and an odd last column tile): ktilde goes to TMEM and the pair MMA reads it
  // there (TS form) -- TMEM has room for one accumulator plus the A ring; NC = 2 needs all 512
  // columns for the two accumulators, so A goes to shared memory (SS form)
  const bool ats = NC == 1;
  const int nst = p1_stages(NC);
  const uint32_t acol0 = (uint32_t)NZ;                   // TMEM A ring (ats): columns [NZ, NZ + nst A1C)
  const size_t a_bytes = ats ? 0 : (size_t)128 * KT1 * 2 * 2;  // A hi | lo of this CTA's 128 rows (smem)
  const size_t bh_bytes = (size_t)(NZ / 2) * KT1 * 2;    // B hi (or lo) of this CTA's NZ/2 columns
  const size_t st_bytes = a_bytes + (size_t)NC * 2 * bh_bytes;
  const size_t x_bytes = (size_t)KT1 * AUXW * 4;         // aux rows of one tile
  uint8_t* ssm = sm;                                     // nst x (A hi | A lo | [B hi | B lo] x NC)
  uint8_t* xsm = ssm + (size_t)nst * st_bytes;           // STA x aux
  uint64_t* full_a = sh.full_a;
  uint64_t* full_b = sh.full_b;
  uint64_t* pfull_b = sh.pfull_b;
  uint64_t* empty = sh.empty;
  uint64_t* full_x = sh.full_x;
  uint64_t* empty_x = sh.empty_x;
  uint64_t& done = sh.done;
  float (*hsum)[128][1 + D] = sh.hsum;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t rank = tc::cluster_rank();  // 0: leader (issues the pair MMAs), 1: peer
  const int row0 = bx * 128;
  const int split = bz;
  const int t_begin = split * a.tiles_per_split;
  const int t_end = min(g.nt1, t_begin + a.tiles_per_split);
  const int ntile = max(0, t_end - t_begin);
  const uint8_t* mtiles = a.tiles + (size_t)m * a.m_stride;  // [ct][t] tiles of output m

  if (tid == 0) stamp(a.dbg, 0);
  if (tid == 0) {
    for (int s = 0; s < ST1; ++s) {
      tc::mbar_init(&full_a[s], 2 * GEN_WARPS);  // the leader's: every generator warp of both CTAs
      tc::mbar_init(&full_b[s], 1);
      tc::mbar_init(&pfull_b[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < STA; ++s) {
      tc::mbar_init(&full_x[s], 1);
      tc::mbar_init(&empty_x[s], 32 * GEN_WARPS);
    }
    tc::mbar_init(&done, 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  tc::cluster_sync();  // both CTAs' barriers exist before any remote arrival or multicast commit
  tc::tc_fence_after();
  pdl_launch_dependents();
  // the operand tiles are static (cache build): the producers start now; everything that reads
  // the previous kernel's outputs (x*) or writes this step's outputs waits for it first
  if (warp >= CTRL_WARPS) pdl_wait();

  if (warp == 0) {
    // ------------------------------------------------ B producer: this CTA's half of each column tile
    if (lane == 0) {
      for (int i = 0; i < ntile; ++i) {
        const int s = i % nst;
        tc::mbar_wait(&empty[s], ((uint32_t)(i / nst) & 1u) ^ 1u);
        tc::mbar_arrive_expect_tx(&full_b[s], (uint32_t)(NC * 2 * bh_bytes));
        uint8_t* dst = ssm + (size_t)s * st_bytes + a_bytes;
        for (int c = 0; c < NC; ++c) {
          // packed tile = [B hi: NZ x KT1 | B lo | aux]; this CTA's NZ/2 columns are the rank-th half
          const uint8_t* src = mtiles + ((size_t)(ct0 + c) * g.nt1 + t_begin + i) * g.t1_bytes;
          tc::bulk_g2s(dst + (size_t)c * 2 * bh_bytes, src + rank * bh_bytes, (uint32_t)bh_bytes, &full_b[s]);
          tc::bulk_g2s(dst + (size_t)c * 2 * bh_bytes + bh_bytes, src + 2 * bh_bytes + rank * bh_bytes,
                       (uint32_t)bh_bytes, &full_b[s]);
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------ aux producer (runs up to STA tiles ahead)
    if (lane == 0) {
      const uint8_t* t0 = mtiles + ((size_t)ct0 * g.nt1 + t_begin) * g.t1_bytes + (size_t)4 * NZ * KT1;
      for (int i = 0; i < ntile; ++i) {
        const int x = i % STA;
        tc::mbar_wait(&empty_x[x], ((uint32_t)(i / STA) & 1u) ^ 1u);
        tc::mbar_arrive_expect_tx(&full_x[x], (uint32_t)x_bytes);
        tc::bulk_g2s(xsm + (size_t)x * x_bytes, t0 + (size_t)i * g.t1_bytes, (uint32_t)x_bytes, &full_x[x]);
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ------------------------------------------------ MMA issuer (the leader): the warp waits,
      // one elected lane issues each tile's 6 NC MMAs back to back
      const uint32_t idesc = tc::idesc_f16(256, NZ);
      constexpr uint32_t SBO = (KT1 / 8) * 128;
      for (int i = 0; i < ntile; ++i) {
        const int s = i % nst;
        const uint32_t ph = (uint32_t)(i / nst) & 1u;
        tc::mbar_wait(&full_b[s], ph);
        tc::mbar_wait(&pfull_b[s], ph);
        tc::mbar_wait(&full_a[s], ph);
        tc::tc_fence_after();
        const uint32_t sbase = tc::smem_u32(ssm + (size_t)s * st_bytes);
        const uint64_t dahi = tc::umma_desc(sbase, 128, SBO);
        const uint64_t dalo = tc::umma_desc(sbase + (uint32_t)(a_bytes / 2), 128, SBO);
        const uint32_t tahi = tmem + acol0 + (uint32_t)(s * A1C), talo = tahi + (uint32_t)(KT1 / 2);
        if (tc::elect_one()) {
          if (!(a.diag & 2)) {
            if (ats) {
#pragma unroll
              for (int ks = 0; ks < KT1 / 16; ++ks) {
                const uint64_t o = (uint64_t)(ks * 16);  // 256 bytes >> 4, start-address field
                const uint32_t ac = (uint32_t)(ks * 8);  // 16 K elements = 8 TMEM columns
                const uint32_t acc0 = (i > 0 || ks > 0) ? 1u : 0u;
                const uint64_t dbhi = tc::umma_desc(sbase, 128, SBO), dblo = tc::umma_desc(sbase + (uint32_t)bh_bytes, 128, SBO);
                tc::mma_f16_ts2(tmem, tahi + ac, dbhi + o, idesc, acc0);
                tc::mma_f16_ts2(tmem, tahi + ac, dblo + o, idesc, 1u);
                tc::mma_f16_ts2(tmem, talo + ac, dbhi + o, idesc, 1u);
              }
            } else {
#pragma unroll
              for (int ks = 0; ks < KT1 / 16; ++ks) {
                const uint64_t o = (uint64_t)(ks * 16);
                const uint32_t acc0 = (i > 0 || ks > 0) ? 1u : 0u;
                for (int c = 0; c < NC; ++c) {
                  const uint32_t bb = sbase + (uint32_t)(a_bytes + (size_t)c * 2 * bh_bytes);
                  const uint64_t dbhi = tc::umma_desc(bb, 128, SBO), dblo = tc::umma_desc(bb + (uint32_t)bh_bytes, 128, SBO);
                  const uint32_t d = tmem + (uint32_t)(c * NZ);
                  tc::mma_f16_2(d, dahi + o, dbhi + o, idesc, acc0);
                  tc::mma_f16_2(d, dahi + o, dblo + o, idesc, 1u);
                  tc::mma_f16_2(d, dalo + o, dbhi + o, idesc, 1u);
                }
              }
            }
          }
          tc::umma_commit2_mc(&empty[s], 3);
        }
        __syncwarp();
        if (i == 0 && lane == 0) stamp(a.dbg, 1);
      }
      if (tc::elect_one()) tc::umma_commit2_mc(&done, 3);
      __syncwarp();
      if (lane == 0) stamp(a.dbg, 2);
    } else if (lane == 0) {
      // ------------------------------------------------ the peer forwards "my B half of stage s landed"
      for (int i = 0; i < ntile; ++i) {
        const int s = i % nst;
        tc::mbar_wait(&full_b[s], (uint32_t)(i / nst) & 1u);
        tc::mbar_arrive_remote(&pfull_b[s], 0);
      }
    }
  } else {
    // ------------------------------------------------ ktilde generators (4 threads per row, 8 n each)
    // warp w serves TMEM lane quarter w % 4 (row r = 32 (w % 4) + lane); qd = which 8 of the 32
    // points; the A tile is written to shared memory as the canonical K-major SS operand
    const int gt = tid - 32 * CTRL_WARPS;  // 0..511
    const int r = (warp % 4) * 32 + lane, qd = (warp - CTRL_WARPS) / 4;
    const int row = row0 + r;
    const uint32_t tlane = (uint32_t)((warp % 4) * 32) << 16;
    // element (r, 8 qd .. 8 qd + 7) of the canonical layout: one 16-byte chunk
    const uint32_t aoff = (uint32_t)((((r >> 3) * (KT1 / 8) + qd) << 6) + ((r & 7) << 3)) * 2u;
    // exponent as (x*_c - X_nc) * kappa / l_c: difference first, then scale (4x smaller fp32
    // error in ktilde than scaling first, scripts/fp32_floor.py)
    float xq[D], sc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      xq[c] = row < a.B ? a.xstar[(size_t)row * D + c] : 0.0f;
      sc[c] = a.qscale[m][c];
    }
    // mean columns, two partial sums per column (even / odd training points: one FFMA2 lane each)
    float2 hacc2[1 + D];
#pragma unroll
    for (int c = 0; c <= D; ++c) hacc2[c] = make_float2(0.0f, 0.0f);
    // the mean columns belong to the column-tile pair ctp = 0 only (C4 / C5 run a single pair: k =
    // 512 is two column tiles)
    auto gen_tiles = [&](auto mean_tag) {
    constexpr bool MEAN = decltype(mean_tag)::value;
    for (int i = 0; i < ntile; ++i) {
      const int s = i % nst, x = i % STA;
      tc::mbar_wait(&full_x[x], (uint32_t)(i / STA) & 1u);               // aux rows of tile i landed
      tc::mbar_wait(&empty[s], ((uint32_t)(i / nst) & 1u) ^ 1u);        // the pair's MMAs released stage s
      const float* aux = reinterpret_cast<const float*>(xsm + (size_t)x * x_bytes);
      uint32_t hw[4], lw[4];
      if (!(a.diag & 1))
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        // training points e and e + 1 of this thread's 8 as the two lanes of fp32x2 operations
        float2 an[NAUX];
        load_aux2<NAUX>(aux + ((qd * 8 + e) >> 1) * (2 * AUXW), an);
        float2 q = make_float2(0.0f, 0.0f), dx[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          dx[c] = sub2(make_float2(xq[c], xq[c]), an[c]);  // x*_c - X_nc
          const float2 df = mul2(dx[c], make_float2(sc[c], sc[c]));
          q = fma2(df, df, q);
        }
        const float2 kt = make_float2(ex2_approx(-q.x), ex2_approx(-q.y));
        // mean column and the mean Jacobian in difference form: sum_n s k_n alpha_n (x*_c - X_nc)
        // (no x* mu - sum k alpha X_c cancellation between two large sums)
        // mu keeps the fused k * (s alpha) + acc (one rounding per term: the mean is the most
        // cancellation-sensitive output); the Jacobian columns take the rounded product
        if (MEAN) {
          hacc2[0] = fma2(kt, an[D], hacc2[0]);
          const float2 ka = mul2(kt, an[D]);
#pragma unroll
          for (int c = 0; c < D; ++c) hacc2[1 + c] = fma2(ka, dx[c], hacc2[1 + c]);
        }
        const float2 kts = mul2(kt, make_float2(SPLIT_UP, SPLIT_UP));  // exact
        const __half2 h2 = __floats2half2_rn(kts.x, kts.y);
        const float2 res = sub2(kts, __half22float2(h2));
        const __half2 l2 = __floats2half2_rn(res.x, res.y);
        hw[e / 2] = *reinterpret_cast<const uint32_t*>(&h2);
        lw[e / 2] = *reinterpret_cast<const uint32_t*>(&l2);
      }
      if (ats) {
        // A tile (row r, K pairs 4 qd .. 4 qd + 3) -> TMEM stage s, hi then lo
        tc::tc_fence_after();
        const uint32_t ta = tmem + tlane + acol0 + (uint32_t)(s * A1C + qd * 4);
        tc::tmem_st4(ta, hw);
        tc::tmem_st4(ta + (uint32_t)(KT1 / 2), lw);
        tc::tmem_st_wait();
        tc::tc_fence_before();
      } else {
        // A tile (row r, K 8 qd .. 8 qd + 7) -> stage s, hi then lo; then make the generic-proxy
        // writes visible to the tensor core (async proxy) before the leader may issue on them
        uint8_t* abase = ssm + (size_t)s * st_bytes;
        *reinterpret_cast<uint4*>(abase + aoff) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(abase + a_bytes / 2 + aoff) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        tc::fence_proxy_async();
      }
      // MEMBAR.CTA: every aux load above has returned before the aux stage is released
      // (SYNCS.ARRIVE does not wait for pending LDS)
      if (!(a.diag & 4)) __threadfence_block();
      tc::mbar_arrive(&empty_x[x]);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(&full_a[s], 0);  // the leader's barrier (both CTAs)
    }
    };
    if (ctp == 0) gen_tiles(std::true_type{});
    else gen_tiles(std::false_type{});
    if (gt == 0) stamp(a.dbg, 3);
    float hacc[1 + D];
#pragma unroll
    for (int c = 0; c <= D; ++c) hacc[c] = hacc2[c].x + hacc2[c].y;
    // ---- mean columns: combine the four quarters of each row (fixed order)
    if (qd > 0)
      for (int c = 0; c <= D; ++c) hsum[qd - 1][r][c] = hacc[c];
    asm volatile("bar.sync 1, %0;" ::"n"(32 * GEN_WARPS) : "memory");
    if (qd == 0 && row < a.B && ctp == 0) {
      float* o = a.P1h + ((size_t)(split * a.m_count + m) * a.B + row) * (1 + D);
      for (int c = 0; c <= D; ++c) o[c] = ((hacc[c] + hsum[0][r][c]) + hsum[1][r][c]) + hsum[2][r][c];
    }
    // ---- z columns: TMEM -> registers -> global (column-major over rows, coalesced)
    tc::mbar_wait(&done, 0);
    __syncwarp();
    tc::tc_fence_after();
    const int quarter = warp % 4;  // TMEM lane quarter accessible to this warp
    const int cg = (warp - CTRL_WARPS) / 4;  // column group 0..3
    const int wrow = quarter * 32 + lane;
    const int gw = cdiv_dev(NZ, 32) * 8;  // columns per group (multiple of 8)
    const int c_begin = cg * gw, c_end = min(NZ, c_begin + gw);
    if (gt == 0) stamp(a.dbg, 4);
    if (FUSED) {
      // partial z tile (nct == 1: NC == 1) -> stage memory [128][NZ + 4] (padded rows: conflict-free
      // v4 stores); the pair's MMAs are complete, so no operand in this memory is still read
      float* zs = reinterpret_cast<float*>(sm) + (size_t)wrow * (NZ + 4);
      for (int c0 = c_begin; c0 < c_end; c0 += 8) {
        float v[8];
        tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, v);
        tc::tmem_ld_wait();
        if (ntile == 0)
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = 0.0f;
        *reinterpret_cast<float4*>(zs + c0) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(zs + c0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
      }
    } else {
      const int grow = row0 + wrow;
      for (int c = 0; c < NC; ++c) {
        float* zout = a.P1z + ((size_t)((split * a.m_count + m) * g.nct + ct0 + c) * NZ) * a.B;
        for (int c0 = c_begin; c0 < c_end; c0 += 8) {
          float v[8];
          tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(c * NZ + c0), v);
          tc::tmem_ld_wait();
          if (grow < a.B) {
#pragma unroll
            for (int u = 0; u < 8; ++u) zout[(size_t)(c0 + u) * a.B + grow] = ntile > 0 ? v[u] : 0.0f;
          }
        }
      }
    }
  }
  if (warp < CTRL_WARPS) pdl_wait();
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // no remote arrival or multicast commit still targets either CTA's barriers
  if (tid == 0) {
    stamp(a.dbg, 5);
    for (int s = 0; s < ST1; ++s) {
      tc::mbar_inval(&full_a[s]);
      tc::mbar_inval(&full_b[s]);
      tc::mbar_inval(&pfull_b[s]);
      tc::mbar_inval(&empty[s]);
    }
    for (int s = 0; s < STA; ++s) {
      tc::mbar_inval(&full_x[s]);
      tc::mbar_inval(&empty_x[s]);
    }
    tc::mbar_inval(&done);
  }
  if (FUSED) {
    const int LDZ = NZ + 4;
    const int rtn = cdiv_dev(a.B, 128);
    const int S = nbz;
    const float* zs = reinterpret_cast<const float*>(sm);
    // CTA (row tile, m, split) finishes rows rr = split, split + S, ... of its tile; the partials
    // of all other rows go to P1z row-major [split][m][row tile][128][NZ] (one warp per row:
    // 512-byte contiguous segments)
    float* dst = a.P1z + ((size_t)(split * a.m_count + m) * rtn + bx) * 128 * NZ;
    for (int rr = warp; rr < 128 && row0 + rr < a.B; rr += THREADS / 32)
      if (rr % S != split)
        for (int c4 = lane; c4 * 4 < NZ; c4 += 32)
          *reinterpret_cast<float4*>(dst + (size_t)rr * NZ + c4 * 4) =
              *reinterpret_cast<const float4*>(zs + rr * LDZ + c4 * 4);
    if (tid == 0) stamp(a.dbg, 8);
  }
}

// Reduce 1 fused into pass 1 (after the grid barrier that follows p1_main<D, true> of every
// CTA): CTA (bx, by, bz) finishes rows bz, bz + S, ... of row tile bx, output m = by: sums the S
// partials in split order, then v = s - ||z||^2, sigma, J^mu, the row scale and the packed Z.
// jmu / sig: this step's rows of the tapes (nullable).
template <int D>
__device__ __forceinline__ void p1_reduce(const P1Args& a, const int bx, const int by, const int bz, const int S,
                                          const uint8_t* sm, float* jmu, float* sig) {
  const Geo& g = a.g;
  const int NZ = g.NZ;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int row0 = bx * 128;
  const int m = by, split = bz;
  const int LDZ = NZ + 4;
  const int rtn = cdiv_dev(a.B, 128);
  const float* zs = reinterpret_cast<const float*>(sm);
  {
    // lane l owns columns 4l .. 4l+3 and 128 + 4l .. 128 + 4l + 3: every float4 load of a warp is
    // one contiguous 512-byte segment (full 32-byte sectors; the L2-only loads are not re-fetched)
    const bool act0 = lane * 4 < NZ, act1 = 128 + lane * 4 < NZ;
    const size_t sstride = (size_t)a.m_count * rtn * 128 * NZ;  // floats per split
    for (int rr = split + S * warp; rr < 128 && row0 + rr < a.B; rr += S * (THREADS / 32)) {
      const int mm = m, row = row0 + rr;
      const float* src = a.P1z + ((size_t)mm * rtn * 128 + row) * NZ + lane * 4;
      const float* own = zs + rr * LDZ + lane * 4;
      const float* hsrc = a.P1h + ((size_t)mm * a.B + row) * (1 + D) + min(lane, D);
      const size_t hstride = (size_t)a.m_count * a.B * (1 + D);
      // sum the S partials in split order (own one from shared memory; 6 splits' loads in flight)
      float z[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) z[e] = 0.0f;
      float hv = 0.0f;
      for (int s0 = 0; s0 < S; s0 += 6) {
        float4 q[6][2];
        float hq[6];
#pragma unroll
        for (int ss = 0; ss < 6; ++ss) {
          if (s0 + ss < S) {
            const bool mine = s0 + ss == split;
            const float* p = src + (s0 + ss) * sstride;
            q[ss][0] = make_float4(0.f, 0.f, 0.f, 0.f);
            q[ss][1] = q[ss][0];
            if (act0) q[ss][0] = mine ? *reinterpret_cast<const float4*>(own) : __ldcg(reinterpret_cast<const float4*>(p));
            if (act1)
              q[ss][1] = mine ? *reinterpret_cast<const float4*>(own + 128) : __ldcg(reinterpret_cast<const float4*>(p + 128));
            if (lane <= D) hq[ss] = __ldcg(hsrc + (s0 + ss) * hstride);
          }
        }
#pragma unroll
        for (int ss = 0; ss < 6; ++ss) {
          if (s0 + ss < S) {
            z[0] += q[ss][0].x; z[1] += q[ss][0].y; z[2] += q[ss][0].z; z[3] += q[ss][0].w;
            z[4] += q[ss][1].x; z[5] += q[ss][1].y; z[6] += q[ss][1].z; z[7] += q[ss][1].w;
            if (lane <= D) hv += hq[ss];
          }
        }
      }
      if (tid == 0) stamp(a.dbg, 9);
      // column scales undone; ||z||^2 (fp64) and max|z| over the row
      double zz = 0.0;
      float zm = 0.0f;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = (e < 4 ? 0 : 128) + lane * 4 + (e & 3);
        const float v = j < g.k ? z[e] * a.colscale[(size_t)mm * g.k + j] : 0.0f;
        z[e] = v;
        zz += (double)v * (double)v;
        zm = fmaxf(zm, fabsf(v));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        zz += __shfl_xor_sync(0xffffffffu, zz, o);
        zm = fmaxf(zm, __shfl_xor_sync(0xffffffffu, zm, o));
      }
      float inv;
      const float sc = pow2_scale_for(zm, &inv) * SPLIT_UP;
      inv *= SPLIT_DOWN;
      const float h0 = __shfl_sync(0xffffffffu, hv, 0);
      const float v = (float)((double)a.s[mm] - zz);
      if (tid == 0) stamp(a.dbg, 10);
      if (lane == 0) {
        const float sg = sqrtf(fmaxf(v, BAGEL_VAR_FLOOR));
        a.zrow_inv[(size_t)mm * a.B + row] = inv;
        a.mu[(size_t)mm * a.B + row] = h0;
        a.var[(size_t)mm * a.B + row] = v;
        if (sig) sig[(size_t)row * g.p + mm] = v > BAGEL_VAR_FLOOR ? sg : -sg;
      }
      if (jmu && lane >= 1 && lane <= D)
        jmu[((size_t)row * g.p + mm) * D + lane - 1] =
            -hv * a.ell2inv[mm][lane - 1];  // J^mu_c = -(1/l_c^2) sum_n s k alpha (x*_c - X_nc)
      // packed pass-2 A operand (see k_r1b_tc): columns 4l.. of group l/2 (half l%2) and
      // 128+4l.. of group 16 + l/2; lo groups follow the KJ/8 hi groups
      const int rrow = row % 128;
      uint8_t* base = a.Zp + ((size_t)mm * rtn + row / 128) * (size_t)128 * g.KJ * 2 * 2;
#pragma unroll
      for (int hlf = 0; hlf < 2; ++hlf) {
        if (hlf == 0 ? !act0 : !act1) continue;
        uint32_t hw[2], lw[2];
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          const float v0 = z[4 * hlf + e] * sc, v1 = z[4 * hlf + e + 1] * sc;
          const __half2 h2 = __floats2half2_rn(v0, v1);
          const float2 hf = __half22float2(h2);
          const __half2 l2 = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
          hw[e / 2] = *reinterpret_cast<const uint32_t*>(&h2);
          lw[e / 2] = *reinterpret_cast<const uint32_t*>(&l2);
        }
        const int grp = hlf * 16 + lane / 2;
        const size_t off = ((size_t)grp * 128 + rrow) * 16 + (lane & 1) * 8;
        *reinterpret_cast<uint2*>(base + off) = make_uint2(hw[0], hw[1]);
        *reinterpret_cast<uint2*>(base + off + (size_t)(g.KJ / 8) * 128 * 16) = make_uint2(lw[0], lw[1]);
      }
    }
    if (tid == 0) stamp(a.dbg, 7);
  }
}

template <int D, bool FUSED>
__global__ void __launch_bounds__(THREADS, 1) k_p1_tc(P1Args a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ P1Shared<D> sh;
  __shared__ uint32_t tmem_base;
  const int nctp = cdiv_dev(a.g.nct, 2);
  const int NC = min(2, a.g.nct - 2 * ((int)blockIdx.y % nctp));
  uint32_t ncols = 32;
  const int need = NC == 1 ? a.g.NZ + p1_stages(1) * A1C : NC * a.g.NZ;  // NC = 1: + the TMEM A ring
  while ((int)ncols < need) ncols <<= 1;
  if (threadIdx.x / 32 == 1) tc::tmem_alloc2(&tmem_base, ncols);  // the pair's accumulators
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  p1_main<D, FUSED>(a, blockIdx.x, blockIdx.y, blockIdx.z, gridDim.z, sm, sh, tmem_base);
  if (threadIdx.x / 32 == 1) tc::tmem_dealloc2(tmem_base, ncols);
  if (FUSED) {
    grid_barrier(a.gbar, a.err_flag);
    if (threadIdx.x == 0) stamp(a.dbg, 6);
    p1_reduce<D>(a, blockIdx.x, blockIdx.y, blockIdx.z, gridDim.z, sm, a.jmu, a.sig);
  }
}


// ====================================================================== reduce 1
struct R1Args {
  Geo g;
  const float* xstar;
  int B, S1;
  const float* P1z;
  const float* P1h;
  const float* colscale;   // [m][k] 2^e_j
  float s[BAGEL_MAX_P];
  float ell2inv[BAGEL_MAX_P][BAGEL_MAX_D];
  float* Z;                // [m][k][B] fp32 z (after the column scales are undone)
  uint8_t* Zp;             // packed pass-2 A operand [m][rowtile][jt][16-byte group][row][4 words]
  float* zrow_inv;         // [m][B] 2^e_r (undo of the per-row Z scale)
  float* mu;               // [m][B]
  float* var;              // [m][B]
  float* jmu;              // [B][p][d] (nullable)
  float* sig;              // [B][p] (nullable)
};

// Reduce 1 in two launches with ample parallelism (the split partials are L2-resident):
//  r1a  grid (row groups of 32, m, j groups of 32): lane = row, warp = 4 j's; sums the S1
//       partials in split order, writes z (Z[m][j][row], coalesced) and per-(j group, row)
//       partial ||z||^2 (fp64) and max|z|.
//  r1b  grid (row groups of 32, m): per-row totals in j-group order -> v, sigma, J^mu,
//       row scale; packs z as the fp16 hi/lo pass-2 A operand (row-major, the TMEM image).
constexpr int R1_JG = 32;
// lane = 4 consecutive rows (float4 traffic when B % 4 == 0: VEC), warp w = columns jg*32 + 4w .. +3,
// CTA = 128 rows
template <bool VEC>
__device__ __forceinline__ float4 ld4(const float* p, int nrows) {
  if (VEC) return __ldg(reinterpret_cast<const float4*>(p));
  return make_float4(nrows > 0 ? __ldg(p) : 0.f, nrows > 1 ? __ldg(p + 1) : 0.f, nrows > 2 ? __ldg(p + 2) : 0.f,
                     nrows > 3 ? __ldg(p + 3) : 0.f);
}
template <bool VEC>
__global__ void __launch_bounds__(256) k_r1a_tc(R1Args a, double* __restrict__ zz_part, float* __restrict__ zmax_part) {
  const Geo& g = a.g;
  const int m = blockIdx.y, jg = blockIdx.z;
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const int row = blockIdx.x * 128 + lane * 4;  // first of this thread's 4 rows
  const bool ok = row < a.B;
  const int nrows = min(4, a.B - row);
  __shared__ double zz_s[8][128];
  __shared__ float zm_s[8][128];
  float4 z[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) z[u] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int j0 = jg * R1_JG + w * 4;
  if (ok) {
    const float* src[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = min(j0 + u, g.k - 1);
      const int ct = j / g.NZ, jr = j % g.NZ;
      src[u] = a.P1z + ((size_t)(m * g.nct + ct) * g.NZ + jr) * a.B + row;
    }
    const size_t sstride = (size_t)g.p * g.nct * g.NZ * a.B;
    // 4 splits x 4 columns of independent 16-byte loads in flight, summed in split order
    for (int s0 = 0; s0 < a.S1; s0 += 4) {
      float4 v[4][4];
#pragma unroll
      for (int ss = 0; ss < 4; ++ss)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[ss][u] = (s0 + ss < a.S1) ? ld4<VEC>(src[u] + (size_t)(s0 + ss) * sstride, nrows) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int ss = 0; ss < 4; ++ss)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          z[u].x += v[ss][u].x;
          z[u].y += v[ss][u].y;
          z[u].z += v[ss][u].z;
          z[u].w += v[ss][u].w;
        }
    }
  }
  double zz[4] = {0.0, 0.0, 0.0, 0.0};
  float zm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = j0 + u;
    if (j < g.k && ok) {
      const float cs = a.colscale[(size_t)m * g.k + j];
      const float4 v = make_float4(z[u].x * cs, z[u].y * cs, z[u].z * cs, z[u].w * cs);
      float* zd = a.Z + ((size_t)m * g.k + j) * a.B + row;
      if (VEC) {
        *reinterpret_cast<float4*>(zd) = v;
      } else {
        zd[0] = v.x;
        if (nrows > 1) zd[1] = v.y;
        if (nrows > 2) zd[2] = v.z;
        if (nrows > 3) zd[3] = v.w;
      }
      zz[0] += (double)v.x * (double)v.x;
      zz[1] += (double)v.y * (double)v.y;
      zz[2] += (double)v.z * (double)v.z;
      zz[3] += (double)v.w * (double)v.w;
      zm[0] = fmaxf(zm[0], fabsf(v.x));
      zm[1] = fmaxf(zm[1], fabsf(v.y));
      zm[2] = fmaxf(zm[2], fabsf(v.z));
      zm[3] = fmaxf(zm[3], fabsf(v.w));
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    zz_s[w][lane * 4 + e] = zz[e];
    zm_s[w][lane * 4 + e] = zm[e];
  }
  __syncthreads();
  if (threadIdx.x < 128) {
    const int rr = blockIdx.x * 128 + threadIdx.x;
    if (rr < a.B) {
      double t = 0.0;
      float mx = 0.0f;
      for (int i = 0; i < 8; ++i) {  // column order within the group: fixed
        t += zz_s[i][threadIdx.x];
        mx = fmaxf(mx, zm_s[i][threadIdx.x]);
      }
      const int njg = cdiv_dev(g.k, R1_JG);
      zz_part[((size_t)m * njg + jg) * a.B + rr] = t;
      zmax_part[((size_t)m * njg + jg) * a.B + rr] = mx;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256) k_r1b_tc(R1Args a, const double* __restrict__ zz_part,
                                                const float* __restrict__ zmax_part) {
  const Geo& g = a.g;
  const int m = blockIdx.y;
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const int row = blockIdx.x * 32 + lane;
  const bool ok = row < a.B;
  __shared__ float scale_s[32];
  __shared__ double t_s[8][32];
  __shared__ float mx_s[8][32];
  __shared__ double lv_s[32][33];  // nct == 1: the fused reduce's 32 "lane values" of ||z||^2, per row
  {
    // warp w: j groups w, w+8, ... (max|z|; ||z||^2 partials when nct > 1)
    const int njg = cdiv_dev(g.k, R1_JG);
    double t = 0.0;
    float mx = 0.0f;
    if (ok) {
      for (int i = w; i < njg; i += 8) {
        if (g.nct > 1) t += zz_part[((size_t)m * njg + i) * a.B + row];
        mx = fmaxf(mx, zmax_part[((size_t)m * njg + i) * a.B + row]);
      }
      if (g.nct == 1) {
        // ||z||^2 in EXACTLY the order of the fused reduce (p1_reduce), so a row's variance does not
        // depend on which of the two paths the launch shape selects: "lane value" l = sequential sum
        // of columns 4l..4l+3 then 128+4l..128+4l+3, then an xor butterfly over the 32 lane values
        for (int l = w; l < 32; l += 8) {
          double zl = 0.0;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = (e < 4 ? 0 : 128) + 4 * l + (e & 3);
            const float v = j < g.k ? a.Z[((size_t)m * g.k + j) * a.B + row] : 0.0f;
            zl += (double)v * (double)v;
          }
          lv_s[l][lane] = zl;
        }
      }
    }
    t_s[w][lane] = t;
    mx_s[w][lane] = mx;
  }
  __syncthreads();
  if (w == 0) {
    float sc = 1.0f;
    if (ok) {
      double t = 0.0;
      float mx = 0.0f;
      for (int i = 0; i < 8; ++i) {  // fixed order
        t += t_s[i][lane];
        mx = fmaxf(mx, mx_s[i][lane]);
      }
      if (g.nct == 1) {
        double v[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) v[l] = lv_s[l][lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          double nv[32];
#pragma unroll
          for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ o];
#pragma unroll
          for (int l = 0; l < 32; ++l) v[l] = nv[l];
        }
        t = v[0];
      }
      // mean columns: the S1 split partials in split order (as p1_reduce)
      float h[1 + D];
#pragma unroll
      for (int c = 0; c <= D; ++c) h[c] = 0.0f;
      for (int s = 0; s < a.S1; ++s) {
        const float* src = a.P1h + ((size_t)(s * g.p + m) * a.B + row) * (1 + D);
#pragma unroll
        for (int c = 0; c <= D; ++c) h[c] += src[c];
      }
      float inv;
      sc = pow2_scale_for(mx, &inv) * SPLIT_UP;
      a.zrow_inv[(size_t)m * a.B + row] = inv * SPLIT_DOWN;
      const float v = (float)((double)a.s[m] - t);
      const float sg = sqrtf(fmaxf(v, BAGEL_VAR_FLOOR));
      a.mu[(size_t)m * a.B + row] = h[0];
      a.var[(size_t)m * a.B + row] = v;
      if (a.sig) a.sig[(size_t)row * g.p + m] = v > BAGEL_VAR_FLOOR ? sg : -sg;
      if (a.jmu)
#pragma unroll
        for (int c = 0; c < D; ++c)
          a.jmu[((size_t)row * g.p + m) * D + c] = -h[1 + c] * a.ell2inv[m][c];
    }
    scale_s[lane] = sc;
  }
  __syncthreads();
  if (!ok) return;
  const float sc = scale_s[lane];
  const int rt = row / 128, rr = row % 128;
  const size_t tile_halfs = (size_t)128 * g.KJ;
  for (int c8 = w; c8 * 8 < g.k; c8 += 8) {
    const int j8 = c8 * 8;
    const int jt = j8 / g.KJ, jr = j8 % g.KJ;
    // the TMEM image of the pass-2 A operand: per row KJ words [hi: KJ/2 | lo: KJ/2] (2 fp16 each),
    // stored as 16-byte groups of 4 words, group-major then row: [group][row 128][4 words], so a
    // warp's load of one group for 32 consecutive rows is one contiguous 512-byte segment
    uint8_t* base = a.Zp + (((size_t)m * cdiv_dev(a.B, 128) + rt) * g.njt + jt) * tile_halfs * 2 * 2;
    uint8_t* zhi = base + ((size_t)(jr / 8) * 128 + rr) * 16;
    uint8_t* zlo = base + ((size_t)(g.KJ / 8 + jr / 8) * 128 + rr) * 16;
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const float v0 = j8 + e < g.k ? a.Z[((size_t)m * g.k + j8 + e) * a.B + row] * sc : 0.0f;
      const float v1 = j8 + e + 1 < g.k ? a.Z[((size_t)m * g.k + j8 + e + 1) * a.B + row] * sc : 0.0f;
      const __half2 h2 = __floats2half2_rn(v0, v1);
      const float2 hf = __half22float2(h2);
      const __half2 l2 = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
      hw[e / 2] = *reinterpret_cast<const uint32_t*>(&h2);
      lw[e / 2] = *reinterpret_cast<const uint32_t*>(&l2);
    }
    *reinterpret_cast<uint4*>(zhi) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(zlo) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
}

// ====================================================================== pass 2
struct P2Args {
  Geo g;
  int m_count;
  const float* xstar;
  int B;
  const uint8_t* tiles;     // [m][jt][t] pass-2 tiles
  size_t m_stride;
  const uint8_t* Zp;        // packed Z
  const float* zrow_inv;    // [m][B]
  int tiles_per_split;
  float* P2;                // [split * njt + jt][m][B][P2_LD]
  float qscale[BAGEL_MAX_P][BAGEL_MAX_D];
  unsigned long long* dbg;  // nullable: per-CTA %globaltimer event stamps (16 per CTA)
  // EPI: the step epilogue fused in after a grid barrier (cooperative launch)
  unsigned long long* gbar;
  EpiArgs e;
};

// EPI (cooperative launch, every CTA resident): after its tiles, each CTA's control warps stage
// theta^T in the idle stage memory while the epilogue warps finish; after a grid barrier (all
// pass-2 partials written), warp w of CTA c runs the step epilogue (policy_rows.cuh) of rows
// c * R + w, ... (R = ceil(B / CTAs)) -- the separate epilogue launch disappears.
template <int D>
struct P2Shared {
  uint64_t zready[4], full_s[ST2], pfull_s[ST2], empty_s[ST2], full_x[STX2], empty_x[STX2], tfull[2], tempty[2],
      mma_done;
  float asum[3][128][1 + D];
};

// Pass 2 of the CTA with grid coordinates (bx, by, bz) (TMEM: 512 columns at `tmem`).  EPI: the
// control warps stage theta^T in the stage memory once every MMA has completed.  Ends with every
// thread past a __syncthreads and the barriers retired.
//
// CTA pairs (cta_group::2): the two CTAs of a cluster along x (row tiles 2c, 2c + 1) run ONE chain
// of M = 256 MMAs issued by the leader (rank 0): each CTA holds its 128 rows of Z in its own TMEM
// (the TS-form A operand) and HALF of every R slab (64 of the tile's 128 training points) in its
// shared memory; each CTA's accumulator receives its own rows x all 128 points.  A pair MMA of
// N = 128 issues at the tensor floor (64.1 cycles per 256 x 128 x 16 vs 108.8 for one CTA's
// 128 x 128 x 16, profiles/r02_b_tc_pair_issue_rate.txt).  Cross-CTA hand-offs: the peer's slab
// loads are forwarded to the leader's pfull_s, both CTAs' epilogue warps arrive on the leader's
// zready / tempty (cluster scope), the leader's commits multicast to both CTAs.
template <int D, bool EPI>
__device__ __forceinline__ void p2_main(const P2Args& a, const int bx, const int by, const int bz, uint8_t* sm,
                                        P2Shared<D>& sh, const uint32_t tmem, const bool stage_theta) {
  const Geo& g = a.g;
  const int KJ = g.KJ;
  const int nsl = KJ / KS2;                            // slabs per tile
  constexpr int NAUX = D + 1;
  constexpr size_t slab_bytes = (size_t)2 * NT2 * KS2;  // this CTA's half (NT2/2 points) of a slab, hi + lo
  constexpr size_t half_bytes = (size_t)NT2 * KS2;      // hi (or lo) of NT2/2 points
  constexpr size_t x_bytes = (size_t)NT2 * AUXW * 4;    // aux rows of one tile
  uint64_t* zready = sh.zready;  // per K slab: that slab's Z columns are in TMEM
  uint64_t* full_s = sh.full_s;
  uint64_t* pfull_s = sh.pfull_s;  // leader: the peer's half of slab s landed
  uint64_t* empty_s = sh.empty_s;
  uint64_t* full_x = sh.full_x;
  uint64_t* empty_x = sh.empty_x;
  uint64_t* tfull = sh.tfull;
  uint64_t* tempty = sh.tempty;
  uint64_t& mma_done = sh.mma_done;
  float (*asum)[128][1 + D] = sh.asum;

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const uint32_t rank = tc::cluster_rank();  // 0: leader (issues the pair MMAs), 1: peer
  const int row0 = bx * 128;
  const bool rows_valid = row0 < a.B;        // the odd-count padding CTA holds no rows
  const int m = by / g.njt, jt = by % g.njt;
  const int split = bz;
  const int t_begin = split * a.tiles_per_split;
  const int t_end = min(g.nt2, t_begin + a.tiles_per_split);
  const int ntile = max(0, t_end - t_begin);
  const uint8_t* tiles = a.tiles + (size_t)m * a.m_stride + ((size_t)jt * g.nt2) * g.t2_bytes;
  uint8_t* ssm = sm;                              // ST2 slab stages
  uint8_t* xsm = ssm + ST2 * slab_bytes;          // STX2 aux stages
  // TMEM columns: [0, 2*NT2) two accumulators, then Z hi (KJ/2 cols) and Z lo (KJ/2 cols)
  constexpr uint32_t ZC = 2 * NT2;

  if (tid == 0) stamp(a.dbg, 0);
  if (tid == 0) {
    // zready / tempty: one arrival per epilogue warp of BOTH CTAs (on the leader's barriers)
    for (int z = 0; z < 4; ++z) tc::mbar_init(&zready[z], 2 * GEN_WARPS);
    for (int s = 0; s < ST2; ++s) {
      tc::mbar_init(&full_s[s], 1);
      tc::mbar_init(&pfull_s[s], 1);
      tc::mbar_init(&empty_s[s], 1);
    }
    for (int s = 0; s < STX2; ++s) {
      tc::mbar_init(&full_x[s], 1);
      tc::mbar_init(&empty_x[s], 32 * GEN_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 2 * GEN_WARPS);
    }
    tc::mbar_init(&mma_done, 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  tc::cluster_sync();  // both CTAs' barriers exist before any remote arrival or multicast commit
  tc::tc_fence_after();
  if (tid == 0) stamp(a.dbg, 7);
  pdl_launch_dependents();
  // operand tiles are static: producers start now; Z / x* readers wait for the previous kernel
  if (warp >= CTRL_WARPS) pdl_wait();

  if (warp == 0) {
    if (lane == 0) {
      int q = 0;
      for (int i = 0; i < ntile; ++i) {
        const uint8_t* src = tiles + (size_t)(t_begin + i) * g.t2_bytes;
        for (int sl = 0; sl < nsl; ++sl, ++q) {
          const int s = q % ST2;
          tc::mbar_wait(&empty_s[s], ((uint32_t)(q / ST2) & 1u) ^ 1u);
          tc::mbar_arrive_expect_tx(&full_s[s], (uint32_t)slab_bytes);
          // packed slab = [hi: NT2 points x KS2 | lo: same]; this CTA's NT2/2 points are the
          // rank-th half of each (canonical layout: row groups outermost)
          const uint8_t* sp = src + (size_t)sl * 2 * slab_bytes;
          uint8_t* dst = ssm + (size_t)s * slab_bytes;
          tc::bulk_g2s(dst, sp + rank * half_bytes, (uint32_t)half_bytes, &full_s[s]);
          tc::bulk_g2s(dst + half_bytes, sp + 2 * half_bytes + rank * half_bytes, (uint32_t)half_bytes, &full_s[s]);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      for (int i = 0; i < ntile; ++i) {
        const int x = i % STX2;
        tc::mbar_wait(&empty_x[x], ((uint32_t)(i / STX2) & 1u) ^ 1u);
        tc::mbar_arrive_expect_tx(&full_x[x], (uint32_t)x_bytes);
        tc::bulk_g2s(xsm + (size_t)x * x_bytes, tiles + (size_t)(t_begin + i) * g.t2_bytes + (size_t)4 * NT2 * KJ,
                     (uint32_t)x_bytes, &full_x[x]);  // every point's aux: both CTAs' epilogues see all NT2
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---- the leader issues the pair's MMAs (M = 256: its rows and the peer's); the whole warp
      // runs the loop (barrier waits), one elected lane issues each slab's 12 MMAs back to back
      const uint32_t idesc = tc::idesc_f16(256, NT2);
      constexpr uint32_t SBO = (KS2 / 8) * 128u;
      const uint32_t zhi = tmem + ZC, zlo = tmem + ZC + (uint32_t)(KJ / 2);
      if (lane == 0) stamp(a.dbg, 1);
      int q = 0;
      for (int i = 0; i < ntile; ++i) {
        const int b = i & 1;
        tc::mbar_wait(&tempty[b], ((uint32_t)(i / 2) & 1u) ^ 1u);  // both epilogues drained acc b
        tc::tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * NT2);
        for (int sl = 0; sl < nsl; ++sl, ++q) {
          const int s = q % ST2;
          const uint32_t ph = (uint32_t)(q / ST2) & 1u;
          if (i == 0) tc::mbar_wait(&zready[sl], 0);  // both CTAs' Z slab sl is in TMEM
          tc::mbar_wait(&full_s[s], ph);
          tc::mbar_wait(&pfull_s[s], ph);
          tc::tc_fence_after();
          const uint32_t sb = tc::smem_u32(ssm + (size_t)s * slab_bytes);
          const uint64_t dbhi = tc::umma_desc(sb, 128, SBO);
          const uint64_t dblo = tc::umma_desc(sb + (uint32_t)half_bytes, 128, SBO);
          if (tc::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < KS2 / 16; ++ks) {
              const uint64_t o = (uint64_t)(ks * 16);
              const uint32_t ac = (uint32_t)(sl * (KS2 / 2) + ks * 8);
              tc::mma_f16_ts2(d, zhi + ac, dbhi + o, idesc, (sl > 0 || ks > 0) ? 1u : 0u);
              tc::mma_f16_ts2(d, zhi + ac, dblo + o, idesc, 1u);
              tc::mma_f16_ts2(d, zlo + ac, dbhi + o, idesc, 1u);
            }
            tc::umma_commit2_mc(&empty_s[s], 3);
          }
          __syncwarp();
        }
        if (tc::elect_one()) tc::umma_commit2_mc(&tfull[b], 3);
        __syncwarp();
        if (i == 0 && lane == 0) stamp(a.dbg, 2);
      }
      if (tc::elect_one()) tc::umma_commit2_mc(&mma_done, 3);  // single phase: every MMA of the pair has completed
      __syncwarp();
      if (lane == 0) stamp(a.dbg, 3);
    } else if (lane == 0) {
      // ---- the peer forwards "my half of slab s landed" to the leader's pfull_s
      const int nq = ntile * nsl;
      for (int q = 0; q < nq; ++q) {
        const int s = q % ST2;
        tc::mbar_wait(&full_s[s], (uint32_t)(q / ST2) & 1u);
        tc::mbar_arrive_remote(&pfull_s[s], 0);
      }
    }
  } else {
    const int quarter = warp % 4, cg = (warp - CTRL_WARPS) / 4;  // lane quarter, 32-column group
    const int r = quarter * 32 + lane;
    const int row = row0 + r;
    // ---- Z hi/lo of this CTA's rows -> TMEM (8-word chunks dealt round-robin to the column groups)
    {
      const int rt = bx;
      // [group of 4 words][row][4 words] (see k_r1b_tc); this row's group gi is at zrow + gi * 128
      const uint4* zrow = reinterpret_cast<const uint4*>(
          a.Zp + (((size_t)m * cdiv_dev(a.B, 128) + rt) * g.njt + jt) * (size_t)128 * KJ * 2 * 2) + r;
      // every load in flight first; then slab by slab (hi chunk sl, lo chunk nsl + sl of the
      // 8-word chunks w0 = cg * 8 + 32 * chunk) into TMEM, releasing the MMA slab by slab
      uint4 q[4][2][2];
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        if (sl < nsl) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int w0 = cg * 8 + (h ? nsl + sl : sl) * 32;
            // L2 loads (not the read-only path): Z is rewritten every step
            q[sl][h][0] = rows_valid ? __ldcg(zrow + (size_t)(w0 / 4) * 128) : make_uint4(0u, 0u, 0u, 0u);
            q[sl][h][1] = rows_valid ? __ldcg(zrow + (size_t)(w0 / 4 + 1) * 128) : make_uint4(0u, 0u, 0u, 0u);
          }
        }
      }
      if (tid == 32 * CTRL_WARPS) stamp(a.dbg, 8 + (q[0][0][0].x == 0x12345678u));
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        if (sl < nsl) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int w0 = cg * 8 + (h ? nsl + sl : sl) * 32;
            const uint32_t v[8] = {q[sl][h][0].x, q[sl][h][0].y, q[sl][h][0].z, q[sl][h][0].w,
                                   q[sl][h][1].x, q[sl][h][1].y, q[sl][h][1].z, q[sl][h][1].w};
            tc::tmem_st8(tmem + ((uint32_t)(quarter * 32) << 16) + ZC + (uint32_t)w0, v);
          }
          tc::tmem_st_wait();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_remote(&zready[sl], 0);  // the leader's barrier (both CTAs)
        }
      }
      if (tid == 32 * CTRL_WARPS) stamp(a.dbg, 6);
    }
    // ------------------------------------------------ epilogue: sum_n (s w_n) ktilde_n [1 | X_n]
    float xq[D], sc[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      xq[c] = row < a.B ? a.xstar[(size_t)row * D + c] : 0.0f;
      sc[c] = a.qscale[m][c];
    }
    const float zinv = row < a.B ? a.zrow_inv[(size_t)m * a.B + row] : 0.0f;
    float2 acc2[1 + D];  // even / odd columns
#pragma unroll
    for (int c = 0; c <= D; ++c) acc2[c] = make_float2(0.0f, 0.0f);
    for (int i = 0; i < ntile; ++i) {
      const int b = i & 1, x = i % STX2;
      tc::mbar_wait(&tfull[b], (uint32_t)(i / 2) & 1u);
      __syncwarp();
      tc::tc_fence_after();
      float w[32];
      const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * NT2 + cg * 32);
      tmem_ld8(ta, w);
      tmem_ld8(ta + 8, w + 8);
      tmem_ld8(ta + 16, w + 16);
      tmem_ld8(ta + 24, w + 24);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(&tempty[b], 0);  // the leader's barrier (both CTAs)
      tc::mbar_wait(&full_x[x], (uint32_t)(i / STX2) & 1u);
      const float* aux = reinterpret_cast<const float*>(xsm + (size_t)x * x_bytes);
#pragma unroll
      for (int u = 0; u < 32; u += 2) {
        // columns u, u + 1 as the two lanes of fp32x2 operations
        float2 an[NAUX];
        load_aux2<NAUX>(aux + ((cg * 32 + u) >> 1) * (2 * AUXW), an);
        float2 q = make_float2(0.0f, 0.0f), dx[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          dx[c] = sub2(make_float2(xq[c], xq[c]), an[c]);  // x*_c - X_nc
          const float2 df = mul2(dx[c], make_float2(sc[c], sc[c]));
          q = fma2(df, df, q);
        }
        const float2 t = mul2(mul2(make_float2(w[u], w[u + 1]), an[D]), make_float2(ex2_approx(-q.x), ex2_approx(-q.y)));
        acc2[0] = add2(acc2[0], t);
        // difference form: sum_n (s w_n k_n) (x*_c - X_nc)
#pragma unroll
        for (int c = 0; c < D; ++c) acc2[1 + c] = fma2(t, dx[c], acc2[1 + c]);
      }
      __threadfence_block();  // every aux load above has returned before the stage is released
      tc::mbar_arrive(&empty_x[x]);
    }
    if (tid == 32 * CTRL_WARPS) stamp(a.dbg, 4);
    float acc[1 + D];
#pragma unroll
    for (int c = 0; c <= D; ++c) acc[c] = acc2[c].x + acc2[c].y;
    // combine the four column groups of each row (fixed order), undo the Z row scale
    if (cg > 0)
      for (int c = 0; c <= D; ++c) asum[cg - 1][r][c] = acc[c];
    asm volatile("bar.sync 1, %0;" ::"n"(32 * GEN_WARPS) : "memory");
    if (cg == 0 && row < a.B) {
      float* o = a.P2 + (((size_t)(split * g.njt + jt) * a.m_count + m) * a.B + row) * P2_LD;
      for (int c = 0; c <= D; ++c) o[c] = (((acc[c] + asum[0][r][c]) + asum[1][r][c]) + asum[2][r][c]) * zinv;
    }
  }
  if (warp < CTRL_WARPS) pdl_wait();
  if (EPI && warp < CTRL_WARPS && stage_theta) {
    // stage theta^T once every MMA of this CTA has completed (stage memory no longer read)
    // (a dedicated one-phase barrier: waiting on tfull's parity could alias an earlier phase)
    tc::mbar_wait(&mma_done, 0);
    const int n4 = (a.e.P.n_params + 3) / 4;
    const float4* src = reinterpret_cast<const float4*>(a.e.thetaT);
    float4* dst = reinterpret_cast<float4*>(sm);
    for (int i = tid; i < n4; i += 32 * CTRL_WARPS) dst[i] = __ldg(src + i);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // no remote arrival or multicast commit still targets either CTA's barriers
  if (tid == 0) {
    stamp(a.dbg, 5);
    for (int z = 0; z < 4; ++z) tc::mbar_inval(&zready[z]);
    for (int s = 0; s < ST2; ++s) {
      tc::mbar_inval(&full_s[s]);
      tc::mbar_inval(&pfull_s[s]);
      tc::mbar_inval(&empty_s[s]);
    }
    for (int s = 0; s < STX2; ++s) {
      tc::mbar_inval(&full_x[s]);
      tc::mbar_inval(&empty_x[s]);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_inval(&tfull[b]);
      tc::mbar_inval(&tempty[b]);
    }
    tc::mbar_inval(&mma_done);
  }
}

// The step epilogue of rows cta * R + w, ... (R = ceil(B / G)), one warp per row; theta^T is in
// shared memory (staged by p2_main<D, true>).  Runs after a grid barrier.
// PHASE 0: epi_pre, 1: epi_post (same warp, same scratch; rows per warp must fit one pass, i.e.
// R <= warps, which tc_pass2_epi_ok guarantees).
template <int D, int PHASE>
__device__ __forceinline__ void epi_rows(const EpiArgs& e, const int t, const int cta, const int G, uint8_t* sm) {
  const int warp = threadIdx.x / 32;
  const int R = (e.B + G - 1) / G;
  const float* th_s = reinterpret_cast<const float*>(sm);
  float* wbase = reinterpret_cast<float*>(sm) + ((e.P.n_params + 3) & ~3) +
                 (size_t)warp * (2 * BAGEL_MAX_WIDTH + rows::epi_scratch_floats<D, 1>());
  if (warp < R) {
    const int b = cta * R + warp;
    if (b < e.B) {
      if (PHASE == 0) rows::epi_pre<D, 1>(e, t, b, 1, wbase + 2 * BAGEL_MAX_WIDTH);
      else rows::epi_post<D, 1>(e, t, b, 1, th_s, wbase, wbase + 2 * BAGEL_MAX_WIDTH);
    }
  }
}

template <int D, bool EPI>
__global__ void __launch_bounds__(THREADS, 1) k_p2_tc(P2Args a) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ P2Shared<D> sh;
  __shared__ uint32_t tmem_base;
  if (threadIdx.x / 32 == 1) tc::tmem_alloc2(&tmem_base, 512);  // the pair's TMEM, same address in both
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  p2_main<D, EPI>(a, blockIdx.x, blockIdx.y, blockIdx.z, sm, sh, tmem_base, a.e.t + 1 < a.e.T);
  if (threadIdx.x / 32 == 1) tc::tmem_dealloc2(tmem_base, 512);
  if (EPI) {
    // arrive, then the pass-1-only half of this CTA's rows while the other CTAs finish pass 2
    const unsigned long long target = grid_arrive(a.gbar);
    const int G = (int)(gridDim.x * gridDim.y * gridDim.z);
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    epi_rows<D, 0>(a.e, a.e.t, cta, G, sm);
    grid_wait(a.gbar, target, a.e.err_flag);
    if (threadIdx.x == 0) stamp(a.dbg, 9);
    epi_rows<D, 1>(a.e, a.e.t, cta, G, sm);
    if (threadIdx.x == 0) stamp(a.dbg, 10);
  }
}

}  // namespace tcg

// ====================================================================== host side
using namespace tcg;

namespace {

#define DISPATCH_D(dv, ...)                              \
  switch (dv) {                                          \
    case 2: { constexpr int D = 2; __VA_ARGS__; break; } \
    case 3: { constexpr int D = 3; __VA_ARGS__; break; } \
    case 4: { constexpr int D = 4; __VA_ARGS__; break; } \
    case 5: { constexpr int D = 5; __VA_ARGS__; break; } \
    case 6: { constexpr int D = 6; __VA_ARGS__; break; } \
    case 7: { constexpr int D = 7; __VA_ARGS__; break; } \
    case 8: { constexpr int D = 8; __VA_ARGS__; break; } \
    default: break;                                      \
  }

Geo geo_of(const bagel_ctx* c) { return make_geo(c->N, c->d, c->p, c->k); }

size_t p1_smem(const Geo& g) {
  // stage ring (A | NC B halves) + aux ring; the FUSED tail parks a [128][NZ + 4] fp32 partial tile
  // in the same memory
  const int NC = g.nct > 1 ? 2 : 1;
  const size_t st = (NC > 1 ? (size_t)128 * KT1 * 4 : 0) + (size_t)NC * g.NZ * KT1 * 2;
  const size_t ring = (size_t)p1_stages(NC) * st + (size_t)STA * KT1 * AUXW * 4;
  return std::max(ring, (size_t)128 * (g.NZ + 4) * 4);
}
size_t p2_smem(const Geo& g) {
  (void)g;
  return (size_t)ST2 * 2 * NT2 * KS2 + (size_t)STX2 * NT2 * AUXW * 4;  // half slabs (CTA pairs)
}

}  // namespace

size_t tc_tiles1_bytes(const bagel_ctx* c) {
  const Geo g = geo_of(c);
  return (size_t)g.nct * g.nt1 * g.t1_bytes;  // per output
}
size_t tc_tiles2_bytes(const bagel_ctx* c) {
  const Geo g = geo_of(c);
  return (size_t)g.njt * g.nt2 * g.t2_bytes;
}
bool tc_supported(const bagel_ctx* c) {
  const Geo g = geo_of(c);
  return p1_smem(g) <= 220 * 1024 && p2_smem(g) <= 220 * 1024;
}

// Pack output m of the cache into the tensor-core operand tiles (cache-build time).
int tc_pack(bagel_ctx* c, int m, cudaStream_t st) {
  const Geo g = geo_of(c);
  TcState& T = c->tcs;
  const double s = (double)c->s[m];
  float* qs_dev = T.qscale + (size_t)m * BAGEL_MAX_D;
  cudaMemcpyAsync(qs_dev, c->gp.qscale[m], sizeof(float) * BAGEL_MAX_D, cudaMemcpyHostToDevice, st);
  const double* R = c->R64 + (size_t)m * c->k * c->N;
  k_colscale<<<c->k, 256, 0, st>>>(R, c->N, c->k, s, T.colscale_inv + (size_t)m * c->k, T.colscale + (size_t)m * c->k);
  k_pack1<<<dim3(g.nt1, g.nct), 256, 0, st>>>(g, c->X, c->alpha64 + (size_t)m * c->N, R, s, qs_dev,
                                              T.colscale_inv + (size_t)m * c->k, T.tiles1 + (size_t)m * T.t1_stride);
  k_pack2<<<dim3(g.nt2, g.njt), 256, 0, st>>>(g, c->X, R, s, qs_dev, T.tiles2 + (size_t)m * T.t2_stride);
  return 3;
}


// N splits of both passes.  The split boundaries depend on N ONLY (never on B or the launch
// shape), so every trajectory's arithmetic -- which training points share a TMEM accumulation
// chain, and the order in which the split partials are summed -- is the same whether it runs in
// a batch of 1 or 65,536, on one GPU or as one shard of eight: per-trajectory results are bitwise
// batch-invariant (tests/test_gpu_parity.py::test_batch_invariance_bitwise).  N is cut into about
// SPLIT_TARGET ranges (the C2 shape -- 8 row tiles x 2 outputs x 9 splits -- fills the 148 SMs in
// one wave), each at most P1_MAX_TILES pass-1 tiles long: the tensor core's fp32 accumulation error
// grows with the chain length (measured: the whole N = 50,000 in one chain put ||z||^2 off by
// 4e-4 s, 1.5x the fp32 tolerance).  With nct == 1 and a one-wave grid, reduce 1
// runs inside pass 1 after a grid barrier (k_p1_tc<D, true>); it sums in exactly the order of the
// separate reduce kernels.  BAGEL_P1_FUSED=0 forces the separate reduce launches.
constexpr int SPLIT_TARGET = 9;
void tc_choose_splits(const bagel_ctx* c, int B, int* S1, int* S2, int* tps1, int* tps2, int* p1_fused) {
  const Geo g = geo_of(c);
  int max_tiles = P1_MAX_TILES;
  if (const char* e = getenv("BAGEL_P1_MAX_TILES")) max_tiles = std::max(1, atoi(e));  // diagnostics only
  *tps1 = std::min(max_tiles, std::max(1, cdiv(g.nt1, SPLIT_TARGET)));
  *S1 = cdiv(g.nt1, *tps1);
  const char* env = getenv("BAGEL_P1_FUSED");
  *p1_fused = g.nct == 1 && tc_pair_row_tiles(B) * g.p * *S1 <= c->num_sms && !(env && env[0] == '0');
  // pass 2 has no accumulation-chain bound (its TMEM chain runs over j, not N): the split only
  // serves occupancy, which small problems need (C2: 8 row tiles x 2 outputs) and large ones do
  // not -- there every extra split re-reads the CTA's 128 KB Z operand (C5: +6% pass-2 time at 9
  // splits).  Still a function of N alone: about 9 splits at N = 5,000, one from N ~ 46,000 up.
  const int s2 = std::max(1, std::min(SPLIT_TARGET, (SPLIT_TARGET * 40) / std::max(1, g.nt2)));
  *tps2 = cdiv(g.nt2, s2);
  *S2 = cdiv(g.nt2, *tps2);
}

size_t tc_p1z_floats(const bagel_ctx* c, int B, int S1) {
  const Geo g = geo_of(c);
  return (size_t)S1 * g.p * g.nct * g.NZ * B;
}
size_t tc_zp_bytes(const bagel_ctx* c, int B) {
  const Geo g = geo_of(c);
  return (size_t)g.p * cdiv(B, 128) * g.njt * 128 * g.KJ * 2 * 2;
}
int tc_njt(const bagel_ctx* c) { return geo_of(c).njt; }
int tc_pair_row_tiles(int B) { return (cdiv(B, 128) + 1) / 2 * 2; }
size_t tc_zpart_count(const bagel_ctx* c, int B) { return (size_t)c->p * cdiv(c->k, R1_JG) * B; }
size_t tc_gbar_count() { return (size_t)GB_STRIDE; }

static void set_attrs() {
  static std::atomic<unsigned long long> devices{0};
  if (!bagel_first_on_device(devices)) return;
  for (int dv = 2; dv <= 8; ++dv) {
    DISPATCH_D(dv, ({
      bagel_set_smem_attr(k_p1_tc<D, false>, 220 * 1024);
      bagel_set_smem_attr(k_p1_tc<D, true>, 220 * 1024);
      bagel_set_smem_attr(k_p2_tc<D, false>, 220 * 1024);
      bagel_set_smem_attr(k_p2_tc<D, true>, 220 * 1024);
    }));
  }
  cudaGetLastError();
}

// The grid-barrier kernels launch WITHOUT the cooperative attribute by default: a cooperative
// launch disables programmatic dependent launch, which costs ~6 us per step at C2 (measured:
// 5.59 vs 6.20 ms per iteration).  Co-residency rests on grid <= #SM x occupancy (checked) and the
// barrier watchdog.  BAGEL_COOP=1 restores cooperative launches (no PDL), e.g. when other
// streams share the GPU.
static bool tc_coop_enabled() {
  const char* env = getenv("BAGEL_COOP");
  return env && env[0] == '1';
}

// Programmatic dependent launch of the GP-step kernels (BAGEL_PDL=0 disables).
static bool tc_pdl_enabled() {
  const char* env = getenv("BAGEL_PDL");
  return !(env && env[0] == '0');
}

int tc_pass1(const bagel_ctx* c, const float* xstar, int B, float* jmu_out, float* sig_out, cudaStream_t st) {
  set_attrs();
  const Geo g = geo_of(c);
  const TcState& T = c->tcs;
  P1Args a{};
  a.g = g;
  a.m_count = c->p;
  a.xstar = xstar;
  a.B = B;
  a.tiles = T.tiles1;
  a.m_stride = T.t1_stride;
  a.tiles_per_split = c->ws.tps1;
  {
    const char* dg = getenv("BAGEL_P1_DIAG");
    a.diag = dg ? atoi(dg) : 0;
  }
  a.P1z = T.P1z;
  a.P1h = T.P1h;
  a.dbg = T.dbg1;
  for (int m = 0; m < c->p; ++m)
    for (int j = 0; j < BAGEL_MAX_D; ++j) a.qscale[m][j] = c->gp.qscale[m][j];
  // CTA pairs along the row tiles; a pair covers two z-column tiles
  dim3 grid(tc_pair_row_tiles(B), c->p * cdiv(g.nct, 2), c->ws.S1tc);
  if (c->ws.p1_fused) {
    a.colscale = T.colscale;
    for (int m = 0; m < c->p; ++m) {
      a.s[m] = c->gp.s[m];
      for (int j = 0; j < BAGEL_MAX_D; ++j) a.ell2inv[m][j] = c->gp.ell2inv[m][j];
    }
    a.Zp = T.Zp;
    a.zrow_inv = T.zrow_inv;
    a.mu = c->ws.mu;
    a.var = c->ws.var;
    a.jmu = jmu_out;
    a.sig = sig_out;
    a.P1h = T.P1h;
    a.gbar = T.gbar;
    a.err_flag = c->ws.err_flag;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = p1_smem(g);
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  int na = 0;
  if (tc_pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = 2;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  if (c->ws.p1_fused && tc_coop_enabled()) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  // a launch error is recorded as the last CUDA error (checked by the caller)
  if (c->ws.p1_fused) {
    DISPATCH_D(c->d, ((void)cudaLaunchKernelEx(&cfg, k_p1_tc<D, true>, a)));
  } else {
    DISPATCH_D(c->d, ((void)cudaLaunchKernelEx(&cfg, k_p1_tc<D, false>, a)));
  }
  return 1;
}

int tc_reduce1(const bagel_ctx* c, const float* xstar, int B, float* jmu_out, float* sig_out, cudaStream_t st) {
  if (c->ws.p1_fused) return 0;  // done inside pass 1
  const Geo g = geo_of(c);
  const TcState& T = c->tcs;
  R1Args a{};
  a.g = g;
  a.xstar = xstar;
  a.B = B;
  a.S1 = c->ws.S1tc;
  a.P1z = T.P1z;
  a.P1h = T.P1h;
  a.colscale = T.colscale;
  for (int m = 0; m < c->p; ++m) {
    a.s[m] = c->gp.s[m];
    for (int j = 0; j < BAGEL_MAX_D; ++j) a.ell2inv[m][j] = c->gp.ell2inv[m][j];
  }
  a.Z = c->ws.Z;
  a.Zp = T.Zp;
  a.zrow_inv = T.zrow_inv;
  a.mu = c->ws.mu;
  a.var = c->ws.var;
  a.jmu = jmu_out;
  a.sig = sig_out;
  if (B % 4 == 0)
    k_r1a_tc<true><<<dim3(cdiv(B, 128), c->p, cdiv(c->k, R1_JG)), 256, 0, st>>>(a, T.zz_part, T.zmax_part);
  else
    k_r1a_tc<false><<<dim3(cdiv(B, 128), c->p, cdiv(c->k, R1_JG)), 256, 0, st>>>(a, T.zz_part, T.zmax_part);
  DISPATCH_D(c->d, (k_r1b_tc<D><<<dim3(cdiv(B, 32), c->p), 256, 0, st>>>(a, T.zz_part, T.zmax_part)));
  return 2;
}

// Can the step epilogue run inside pass 2 (cooperative: one resident wave; theta^T and the
// per-warp buffers fit the stage memory)?
bool tc_pass2_epi_ok(const bagel_ctx* c, int B) {
  const Geo g = geo_of(c);
  const long long ctas = (long long)tc_pair_row_tiles(B) * c->p * g.njt * c->ws.S2tc;
  const size_t need = sizeof(float) * (((size_t)c->pol.n_params + 3) / 4 * 4 +
                                       (size_t)(THREADS / 32) * (2 * BAGEL_MAX_WIDTH + rows::epi_scratch_floats<8, 1>()));
  const char* env = getenv("BAGEL_P2_EPI");
  const long long rows_per_cta = ctas > 0 ? (B + ctas - 1) / ctas : 0;
  return ctas <= c->num_sms && need <= p2_smem(g) && rows_per_cta <= THREADS / 32 && !(env && env[0] == '0');
}

int tc_pass2(const bagel_ctx* c, const float* xstar, int B, const EpiArgs* epi, cudaStream_t st) {
  set_attrs();
  const Geo g = geo_of(c);
  const TcState& T = c->tcs;
  P2Args a{};
  a.g = g;
  a.m_count = c->p;
  a.xstar = xstar;
  a.B = B;
  a.tiles = T.tiles2;
  a.m_stride = T.t2_stride;
  a.Zp = T.Zp;
  a.zrow_inv = T.zrow_inv;
  a.tiles_per_split = c->ws.tps2;
  a.P2 = c->ws.P2;
  a.dbg = T.dbg2;
  for (int m = 0; m < c->p; ++m)
    for (int j = 0; j < BAGEL_MAX_D; ++j) a.qscale[m][j] = c->gp.qscale[m][j];
  dim3 grid(tc_pair_row_tiles(B), c->p * g.njt, c->ws.S2tc);  // CTA pairs along the row tiles
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = p2_smem(g);
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  int na = 0;
  at[na].id = cudaLaunchAttributeClusterDimension;
  at[na].val.clusterDim.x = 2;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  if (tc_pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (epi) {
    a.e = *epi;
    a.gbar = T.gbar + tc_gbar_count();  // pass 2's own counters (pass 1 has another grid shape)
    if (tc_coop_enabled()) {
      at[na].id = cudaLaunchAttributeCooperative;
      at[na].val.cooperative = 1;
      ++na;
    }
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (epi) {
    DISPATCH_D(c->d, ((void)cudaLaunchKernelEx(&cfg, k_p2_tc<D, true>, a)));
  } else {
    DISPATCH_D(c->d, ((void)cudaLaunchKernelEx(&cfg, k_p2_tc<D, false>, a)));
  }
  return 1;
}
