// Philox4x32-10 Gumbel-max temperature sampler, device side.
//
// Operation (readings R10/R11; "temperature 0.8",
// Eq. 1 l.120-125 "randomly sampling from the policy"):
//   token = argmax_v fl(fl(z_v * invT) + G_v),  G_v = -log(-log(u_v)),
//   u_v   = (2*(x >> 9) + 1) * 2^-24,  x = Philox4x32-10(key = seed,
//           ctr = (v >> 2, t, uid, 0)) word (v & 3);
//   ties  -> lowest v through the 64-bit key (ord(score) << 32) | ~v.
// Every float op is an explicit round-to-nearest intrinsic so nvcc cannot
// contract or reorder it: the kernel takes the same decision as the CPU
// oracle on identical logits.
#pragma once
#include <cstdint>

namespace isk {

struct Philox4 {
  uint32_t x[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                 uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  Philox4 o;
  o.x[0] = c0;
  o.x[1] = c1;
  o.x[2] = c2;
  o.x[3] = c3;
  return o;
}

__device__ __forceinline__ float uniform_from_bits(uint32_t x) {
  return __fmul_rn(__uint2float_rn(((x >> 9) << 1) | 1u), 5.9604644775390625e-08f /* 2^-24 */);
}

// log(x) for positive normal fp32 x; identical op sequence to oracle/sampler.py:logf_is.
__device__ __forceinline__ float logf_is(float x) {
  const uint32_t b = __float_as_uint(x);
  int e = (int)(b >> 23) - 127;
  float m = __uint_as_float((b & 0x007FFFFFu) | 0x3F800000u);
  if (m > __uint_as_float(0x3FB504F3u)) {
    m = __fmul_rn(m, 0.5f);
    e += 1;
  }
  const float f = __fsub_rn(m, 1.0f);
  const float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
  const float z = __fmul_rn(s, s);
  float p = __fadd_rn(__fmul_rn(z, 2.0f / 9.0f), 2.0f / 7.0f);
  p = __fadd_rn(__fmul_rn(z, p), 2.0f / 5.0f);
  p = __fadd_rn(__fmul_rn(z, p), 2.0f / 3.0f);
  const float r = __fadd_rn(__fmul_rn(__fmul_rn(s, z), p), __fmul_rn(2.0f, s));
  return __fadd_rn(__fmul_rn(__int2float_rn(e), 0.6931471805599453f), r);
}

__device__ __forceinline__ float gumbel(uint64_t seed, uint32_t uid, uint32_t t, uint32_t v) {
  const Philox4 o = philox4x32_10(v >> 2, t, uid, 0u, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint32_t w = o.x[v & 3];
  const float u = uniform_from_bits(w);
  return -logf_is(-logf_is(u));
}

__device__ __forceinline__ uint64_t order_key(float score, uint32_t v) {
  const uint32_t b = __float_as_uint(score);
  const uint32_t o = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((uint64_t)o << 32) | (uint64_t)(0xFFFFFFFFu - v);
}

}  // namespace isk
