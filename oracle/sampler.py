"""Oracle: Gumbel-max temperature sampler on Philox4x32-10.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md l.382 fixes only "temperature of 0.8"; l.122 (Eq. 1) says completions
are sampled from pi_theta.  Everything else is DESIGN.md reading R10/R11:

  token = argmax_v  fl(fl(z_v * invT) + G_v),   invT = fl32(1/T) (= 1.25 for T = 0.8)
  G_v   = -logf_is(-logf_is(u_v))                (Gumbel(0,1) by inversion)
  u_v   = (2*(x >> 9) + 1) * 2^-24               (x = Philox word v & 3)
  x     = Philox4x32-10(key = (seed lo, seed hi),
                        ctr = (v >> 2, t, uid, 0))[v & 3]
  ties  -> lowest v, via the 64-bit key (ord(score) << 32) | (2^32-1-v).

Argmax of z/T + Gumbel noise is an exact draw from softmax(z/T) (the Gumbel-max
trick), so this *is* temperature sampling; the fp32 op sequence is fixed so the
GPU kernel reproduces every decision bit-exactly on identical logits.  All fp32
operations below are single IEEE binary32 ops with round-to-nearest-even; numpy
float32 scalar/array arithmetic is exactly that (no contraction into FMA).

Pins (tests/test_oracle_sampler.py): Random123 Philox KATs, logf_is vs math.log
within 2 ulp, chi-square of sampled frequencies against softmax(z/T), T->0
argmax, tie-break.

top-p < 1 (BASELINE north_star "temperature/top-p sampler";
the paper itself never uses it).  DESIGN.md reading R36, every decision
in exactly reproducible arithmetic:
  u_v = fl(z_v * invT);  e_v = expf_is(fl(u_v - max u))      (fixed fp32 op sequence)
  w_v = floor(e_v * 2^44)  (integer; exact)                   W = sum_v w_v  (exact)
  thr = ceil(fl64(top_p) * fl64(W))                            (binary64 ops)
  order the vocabulary by (-e_v, v); the nucleus is the shortest prefix whose
  integer mass reaches thr; the token is the Gumbel-max key (as above) over the
  nucleus only.  Pins: fp64 nucleus by definition (away from boundaries),
  top_p -> 0 gives the argmax, chi-square against the renormalised nucleus.
"""
import math

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds (Salmon et al., SC'11; Random123 constants).

    ctr: uint32 array [..., 4]; key: (k0, k1) Python ints.  Returns uint32 [..., 4].
    """
    c = np.asarray(ctr, dtype=np.uint64) & _MASK
    c0, c1, c2, c3 = c[..., 0], c[..., 1], c[..., 2], c[..., 3]
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c0          # < 2^64, exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def uniform_from_bits(x):
    """u = (2*(x>>9)+1) * 2^-24, exact in fp32, u in [2^-24, 1-2^-24]."""
    x = np.asarray(x, dtype=np.uint32)
    k = ((x >> np.uint32(9)) << np.uint32(1)) | np.uint32(1)
    return k.astype(np.float32) * np.float32(2.0 ** -24)


_SQRT2 = np.float32(np.uint32(0x3FB504F3).view(np.float32))  # 1.41421354f
_C9 = np.float32(2.0 / 9.0)
_C7 = np.float32(2.0 / 7.0)
_C5 = np.float32(2.0 / 5.0)
_C3 = np.float32(2.0 / 3.0)
_LN2 = np.float32(0.6931471805599453)


def logf_is(x):
    """Natural log of positive normal fp32 x as a FIXED fp32 op sequence.

    log(x) = e*ln2 + log(m), m in [sqrt(2)/2, sqrt(2)];
    log(m) = 2*atanh(s), s = (m-1)/(m+1) = 2s + s*z*(2/3 + z*(2/5 + z*(2/7 + z*2/9))),
    z = s^2 (series truncated after s^9; |s| <= 0.1716).  Every step is one
    separately rounded fp32 op; the GPU side implements the same sequence
    with __f*_rn intrinsics.
    """
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32)
    e = (b >> np.uint32(23)).astype(np.int32) - np.int32(127)
    m = ((b & np.uint32(0x007FFFFF)) | np.uint32(0x3F800000)).view(np.float32)
    big = m > _SQRT2
    m = np.where(big, m * np.float32(0.5), m).astype(np.float32)
    e = np.where(big, e + 1, e)
    f = (m - np.float32(1.0)).astype(np.float32)
    s = (f / (np.float32(2.0) + f)).astype(np.float32)
    z = (s * s).astype(np.float32)
    p = (z * _C9).astype(np.float32) + _C7
    p = (z * p).astype(np.float32) + _C5
    p = (z * p).astype(np.float32) + _C3
    sz = (s * z).astype(np.float32)
    r = ((sz * p).astype(np.float32) + (np.float32(2.0) * s).astype(np.float32)).astype(np.float32)
    ef = e.astype(np.float32)
    return ((ef * _LN2).astype(np.float32) + r).astype(np.float32)


def gumbel_noise(seed, uid, t, vocab):
    """G_v for v in [0, vocab): fp32 array, counter (v>>2, t, uid, 0)."""
    assert vocab % 4 == 0, "vocab must be a multiple of 4 (one Philox call per 4 entries)"
    n = vocab // 4
    ctr = np.zeros((n, 4), dtype=np.uint64)
    ctr[:, 0] = np.arange(n, dtype=np.uint64)
    ctr[:, 1] = t
    ctr[:, 2] = uid
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    words = philox4x32_10(ctr, key).reshape(-1)        # word index = v & 3
    u = uniform_from_bits(words)
    e = -logf_is(u)                                     # Exp(1) draw, > 0
    return -logf_is(e)


def inv_temperature(T):
    return np.float32(1.0 / T)


def score(z, g, invT):
    """fl(fl(z*invT) + g) in fp32."""
    z = np.asarray(z, dtype=np.float32)
    return ((z * np.float32(invT)).astype(np.float32) + g).astype(np.float32)


def order_key(scores):
    """64-bit keys: (ord(score) << 32) | (2^32-1-v); max key = argmax, ties -> lowest v."""
    b = np.asarray(scores, dtype=np.float32).view(np.uint32).astype(np.uint64)
    neg = (b & np.uint64(0x80000000)) != 0
    o = np.where(neg, (~b) & _MASK, b | np.uint64(0x80000000))
    v = np.arange(len(b), dtype=np.uint64)
    return (o << np.uint64(32)) | (_MASK - v)


def sample_token(logits_f32, seed, uid, t, T=0.8):
    """One Gumbel-max draw from softmax(logits/T); logits are fp32 [vocab]."""
    z = np.asarray(logits_f32, dtype=np.float32)
    if not np.all(np.isfinite(z)):
        raise ValueError("non-finite logits")
    g = gumbel_noise(seed, uid, t, len(z))
    k = order_key(score(z, g, inv_temperature(T)))
    return int(np.argmax(k))


def sample_margin(logits_f32, seed, uid, t, T=0.8):
    """(token, top1 score - top2 score): used to classify near-ties in parity."""
    z = np.asarray(logits_f32, dtype=np.float32)
    s = score(z, gumbel_noise(seed, uid, t, len(z)), inv_temperature(T)).astype(np.float64)
    i = int(np.argmax(order_key(s.astype(np.float32))))
    s2 = s.copy()
    s2[i] = -np.inf
    return i, float(s[i] - s2.max())


_LOG2E = np.float32(1.4426950408889634)
_LN2_HI = np.uint32(0x3F317200).view(np.float32)   # 0.693145751953125 (exact products n*_LN2_HI)
_LN2_LO = np.uint32(0x35BFBE8E).view(np.float32)   # ln2 - _LN2_HI
_EXP_C = [np.float32(1.0 / 720.0), np.float32(1.0 / 120.0), np.float32(1.0 / 24.0), np.float32(1.0 / 6.0),
          np.float32(0.5), np.float32(1.0), np.float32(1.0)]


def expf_is(d):
    """exp(d) for fp32 d <= 0 as a FIXED fp32 op sequence (R36): n = rint(d*log2e),
    r = (d - n*ln2_hi) - n*ln2_lo (Cody-Waite), degree-6 Taylor polynomial in Horner
    form, times 2^n; 0 when n < -125.  Every step one separately rounded fp32 op."""
    d = np.asarray(d, dtype=np.float32)
    n = np.rint((d * _LOG2E).astype(np.float32)).astype(np.float32)
    r = (d - (n * _LN2_HI).astype(np.float32)).astype(np.float32)
    r = (r - (n * _LN2_LO).astype(np.float32)).astype(np.float32)
    p = _EXP_C[0]
    for c in _EXP_C[1:]:
        p = ((r * p).astype(np.float32) + c).astype(np.float32)
    ni = n.astype(np.int32)
    ok = ni >= -125
    two_n = ((np.where(ok, ni, 0) + 127).astype(np.uint32) << np.uint32(23)).view(np.float32)
    return np.where(ok, (p * two_n).astype(np.float32), np.float32(0.0)).astype(np.float32)


def topp_nucleus(logits_f32, T, top_p):
    """Boolean mask of the top-p nucleus (R36)."""
    z = np.asarray(logits_f32, dtype=np.float32)
    u = (z * inv_temperature(T)).astype(np.float32)
    e = expf_is((u - u.max()).astype(np.float32))
    w = np.floor((e * np.float32(2.0 ** 44)).astype(np.float32).astype(np.float64)).astype(np.uint64)
    W = int(sum(int(x) for x in w))
    thr = math.ceil(float(np.float32(top_p)) * float(W))
    order = np.lexsort((np.arange(len(z)), -e.astype(np.float64)))   # (-e, v)
    cum = np.cumsum(w[order], dtype=np.uint64)                          # exact: W < 2^63
    k = int(np.searchsorted(cum, np.uint64(thr)))                       # first prefix with mass >= thr
    mask = np.zeros(len(z), dtype=bool)
    mask[order[:k + 1]] = True
    return mask


def sample_token_topp(logits_f32, seed, uid, t, T=0.8, top_p=1.0):
    """Gumbel-max over the top-p nucleus; top_p >= 1 (or <= 0) is the plain sampler."""
    if not 0.0 < top_p < 1.0:
        return sample_token(logits_f32, seed, uid, t, T)
    z = np.asarray(logits_f32, dtype=np.float32)
    k = order_key(score(z, gumbel_noise(seed, uid, t, len(z)), inv_temperature(T)))
    k = np.where(topp_nucleus(z, T, top_p), k, np.uint64(0))
    return int(np.argmax(k))
