// philox.cuh -- counter-based Philox4x32-10 (Salmon et al., SC'11) and the
// Box-Muller map used for every random draw of the hot path and the Lanczos
// restart vectors (north star "(5) counter-based Philox eps indexed by
// (traj, step, dim), so the oracle reproduces every draw").
//
// Convention:
//   key = (seed & 0xffffffff, seed >> 32)
//   rollout ctr = (b_global, t, m >> 2, 0); eps_{b,t,m} = normals[m & 3]
//   restart ctr = (restart_idx, n >> 2, m, 1) with key ("LOVE", 0)
//   u_i = ((o_i >> 9) + 0.5) * 2^-23  (exact in fp32 and fp64)
//   eps = sqrt(-2 ln u0) cos(2 pi u1), sqrt(-2 ln u0) sin(2 pi u1), same for (u2, u3)
#pragma once
#include <stdint.h>

__host__ __device__ __forceinline__ uint4 bagel_philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

__device__ __forceinline__ float bagel_u23(uint32_t o) {
  return (__uint2float_rn(o >> 9) + 0.5f) * 0x1p-23f;
}

// fp32 Box-Muller with accurate logf / sincospif / sqrtf (reading R25: no __logf).
__device__ __forceinline__ float4 bagel_box_muller(uint4 o) {
  const float u0 = bagel_u23(o.x), u1 = bagel_u23(o.y), u2 = bagel_u23(o.z), u3 = bagel_u23(o.w);
  const float r0 = sqrtf(-2.0f * logf(u0)), r1 = sqrtf(-2.0f * logf(u2));
  float s1, c1, s3, c3;
  sincospif(2.0f * u1, &s1, &c1);
  sincospif(2.0f * u3, &s3, &c3);
  return make_float4(r0 * c1, r0 * s1, r1 * c3, r1 * s3);
}

// fp64 variant (Lanczos restart vectors are part of the fp64 cache build).
__device__ __forceinline__ double bagel_u23d(uint32_t o) {
  return ((double)(o >> 9) + 0.5) * 0x1p-23;
}

__device__ __forceinline__ double bagel_normal_d(uint4 o, int which) {
  const double u0 = bagel_u23d(which < 2 ? o.x : o.z);
  const double u1 = bagel_u23d(which < 2 ? o.y : o.w);
  const double r = sqrt(-2.0 * log(u0));
  double sn, cs;
  sincospi(2.0 * u1, &sn, &cs);
  return (which & 1) ? r * sn : r * cs;
}

__device__ __forceinline__ float4 bagel_rollout_eps4(uint64_t seed, uint32_t b_global, uint32_t t) {
  const uint4 o = bagel_philox4x32_10(make_uint4(b_global, t, 0u, 0u), (uint32_t)(seed & 0xffffffffu),
                                      (uint32_t)(seed >> 32));
  return bagel_box_muller(o);
}

__device__ __forceinline__ float bagel_f4get(float4 v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
