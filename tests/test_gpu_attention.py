"""Kernel-level parity of the decode split attention (the core row).

`is_dbg_attn` runs the work list and exactly the launches one decode layer issues
(tcgen05 shared prefix, per-slot paged suffix units, LSE merge; DESIGN R8) on
caller data.  The oracle is the textbook definition (oracle.attention.attention,
PAPER.md §2.1 l.108) over the CONCATENATION [shared prefix; the row's own suffix]
(PAPER.md l.172 the prompt KV is shared, l.205 each sample keeps its own response
KV), in fp64 on the same bf16 inputs.  Tolerance (DESIGN R31 / SURVEY C31): both
sides start from identical bf16 q/K/V and differ only in fp32 accumulation order
(the prefix P enters the MMA as a bf16 hi/lo pair, ~2^-16), so the fp32 output
must be within 1e-4 normwise per (row, head) and max-abs 1e-4 * max|ref|; the bf16
output must be the round-to-nearest-even of the fp32 one; idle rows stay unwritten.

Suffix lengths cover one token, page and chunk boundaries (16/17, 32/33, 64/65),
mid lengths and the >32-partial merge branch (960/961/1023/1024 tokens: more
than 32 partials per row with 32-token units).
"""
import math

import numpy as np
import pytest
import torch

from oracle.attention import attention

pytestmark = pytest.mark.gpu

LENS = [1, 16, 17, 32, 33, 64, 65, 500, 960, 961, 1023, 1024]


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    _lib.load()
    return _lib


def _case(rows, groups, grp_rows, plen, Hq, Hkv, lens, pt=16, max_new=1024, seed=0, qscale=1.0):
    """Random bf16 inputs; row r gets lens[r] suffix tokens (0 = idle) on shuffled pages."""
    gen = torch.Generator().manual_seed(seed)
    maxp = math.ceil(max_new / pt)
    q = (torch.randn(rows, Hq, 128, generator=gen) * qscale).to(torch.bfloat16)
    prefix = torch.randn(groups, 2, Hkv, plen, 128, generator=gen).to(torch.bfloat16)
    need = [math.ceil(n / pt) for n in lens]
    num_pages = sum(need) + 3
    pool = torch.randn(num_pages, 2, Hkv, pt, 128, generator=gen).to(torch.bfloat16)
    perm = torch.randperm(num_pages, generator=gen).tolist()
    pagetab = torch.zeros(rows, maxp, dtype=torch.int32)
    k = 0
    for r, n in enumerate(need):
        for j in range(n):
            pagetab[r, j] = perm[k]
            k += 1
    row_len = torch.tensor(lens, dtype=torch.int32)
    return q, prefix, pool, pagetab, row_len


def _oracle(q, prefix, pool, pagetab, row_len, grp_rows, pt):
    """fp64 softmax attention over [prefix of the row's group; the row's suffix tokens]."""
    rows, Hq, _ = q.shape
    Hkv = prefix.shape[2]
    rep = Hq // Hkv
    q64, pre64, pool64 = q.double().numpy(), prefix.double().numpy(), pool.double().numpy()
    out = {}
    for r in range(rows):
        n = int(row_len[r])
        if n == 0:
            continue
        m = r // grp_rows
        pages = [int(p) for p in pagetab[r, :math.ceil(n / pt)]]
        for h in range(Hkv):
            Ks = np.concatenate([pool64[p, 0, h] for p in pages])[:n]
            Vs = np.concatenate([pool64[p, 1, h] for p in pages])[:n]
            K = np.concatenate([pre64[m, 0, h], Ks])
            V = np.concatenate([pre64[m, 1, h], Vs])
            for e in range(rep):
                out[(r, h * rep + e)] = attention(q64[r, h * rep + e], K, V)
    return out


def _check(lib, rows, groups, grp_rows, plen, Hq, Hkv, lens, impl, seed, qscale=1.0, pt=16):
    q, prefix, pool, pagetab, row_len = _case(rows, groups, grp_rows, plen, Hq, Hkv, lens, seed=seed, qscale=qscale,
                                             pt=pt)
    dev = [t.cuda() for t in (q, prefix, pool, pagetab, row_len)]
    f32 = torch.full((rows, Hq, 128), float("nan"), device="cuda")
    out, _ = lib.is_dbg_attn(*dev, grp_rows=grp_rows, impl=impl, out_f32=f32)
    torch.cuda.synchronize()
    ref = _oracle(q, prefix, pool, pagetab, row_len, grp_rows, pt)
    got, got_bf = f32.cpu().double().numpy(), out.cpu()
    # the bf16 output is the RNE rounding of the fp32 one (r4)
    live = row_len.numpy() > 0
    assert torch.equal(got_bf[live], f32.cpu()[live].to(torch.bfloat16))
    assert torch.count_nonzero(got_bf[~live]) == 0, "idle rows must stay unwritten"
    worst = 0.0
    for (r, qh), o in ref.items():
        g = got[r, qh]
        err = np.linalg.norm(g - o) / np.linalg.norm(o)
        mabs = np.max(np.abs(g - o)) / np.max(np.abs(o))
        worst = max(worst, err)
        assert err < 1e-4 and mabs < 1e-4, (r, qh, int(row_len[r]), err, mabs)
    return worst


def _lens(rows, groups, grp_rows, rot=0):
    """LENS cycled over the groups' rows with every 4th row idle; rows past groups*grp_rows idle."""
    out, k = [], rot
    for r in range(rows):
        if r >= groups * grp_rows or r % 4 == 3:
            out.append(0)
        else:
            out.append(LENS[k % len(LENS)])
            k += 1
    return out


# (rows = row_capacity, groups, rows per group): config 3 (g = 8 in 16 rows), a full 16-row
# group, and the co-resident layouts of NEXT-1 (4 x 8 in 32 rows, 8 x 8 and 2 x 32 in 64 rows)
LAYOUTS = [(16, 1, 8), (16, 1, 16), (32, 4, 8), (64, 8, 8), (64, 2, 32)]


@pytest.mark.parametrize("rows,groups,grp_rows", LAYOUTS)
@pytest.mark.parametrize("plen", [1, 16, 255])
def test_split_attention_default_impl(lib, rows, groups, grp_rows, plen):
    """The launches the decode step uses at this row capacity (impl 0), 1.7B heads (16 q / 8 kv)."""
    lens = _lens(rows, groups, grp_rows, rot=plen)
    _check(lib, rows, groups, grp_rows, plen, 16, 8, lens, 0, seed=rows * 1000 + plen)


@pytest.mark.parametrize("impl", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("rows,groups,grp_rows", [(16, 1, 8), (16, 1, 16), (64, 8, 8)])
def test_split_attention_every_impl(lib, impl, rows, groups, grp_rows):
    """Each launch variant on every layout it serves (1 warp units, 2 CTA units + merge kernel,
    3 = CUDA-core prefix: one group, 4 = mma.sync units; 5 / 6 = 0 / 4 with the query-rows-as-M
    prefix kernel forced instead of the tokens-as-M one)."""
    if impl == 3 and groups > 1:
        pytest.skip("the CUDA-core prefix serves one group")
    lens = _lens(rows, groups, grp_rows, rot=impl)
    _check(lib, rows, groups, grp_rows, 255, 16, 8, lens, impl, seed=impl * 77 + rows)


def test_split_attention_all_long(lib):
    """Every row past 960 tokens (the >32-partial merge branch on every row), peaky scores."""
    lens = [960, 961, 1000, 1023, 1024, 999, 977, 1015] * 2
    _check(lib, 16, 1, 16, 255, 16, 8, lens, 0, seed=5, qscale=3.0)


@pytest.mark.parametrize("Hq,Hkv,grp_rows,rows", [(32, 8, 8, 16), (4, 2, 8, 16), (16, 16, 16, 16), (64, 8, 8, 64)])
def test_split_attention_other_gqa(lib, Hq, Hkv, grp_rows, rows):
    """Other query/kv head ratios: 4B (rep 4), tiny (rep 2, Hkv 2), rep 1, rep 8 (CUDA-core
    prefix at 64 rows: N = 64 x 8 > 64)."""
    groups = 1 if rows == 16 or Hq // Hkv == 8 else rows // grp_rows
    grp = rows if Hq // Hkv == 8 else grp_rows
    lens = _lens(rows, groups, grp, rot=Hq)
    _check(lib, rows, groups, grp, 255, Hq, Hkv, lens, 0, seed=Hq * 3 + Hkv)


def test_split_attention_errors(lib):
    """More partials than the merge holds, and a length past the page table."""
    from paper_2506_22950_b200._lib import InfsampError
    q, prefix, pool, pagetab, row_len = _case(16, 1, 8, 255, 16, 8, [5] * 8 + [0] * 8)
    dev = [t.cuda() for t in (q, prefix, pool, pagetab, row_len)]
    bad_len = dev[4].clone()
    bad_len[0] = 1025
    with pytest.raises(InfsampError):
        lib.is_dbg_attn(dev[0], dev[1], dev[2], dev[3], bad_len, grp_rows=8)
    with pytest.raises(InfsampError):
        lib.is_dbg_attn(*dev, grp_rows=8, impl=7)


@pytest.mark.parametrize("pt", [4, 8, 32, 64])
def test_split_attention_page_sizes(lib, pt):
    """Other page sizes: 8 and 32 take the mma.sync units (one TMA box per page half),
    4 falls back to the warp units, 64 to the 64-token CTA units + merge kernel."""
    lens = _lens(16, 1, 16, rot=pt)
    _check(lib, 16, 1, 16, 255, 16, 8, lens, 0, seed=pt, pt=pt)


@pytest.mark.parametrize("Hq,Hkv,grp_rows,impl", [(16, 8, 64, 0), (32, 8, 64, 0), (32, 8, 32, 0), (16, 8, 64, 3)])
def test_split_attention_large_groups(lib, Hq, Hkv, grp_rows, impl):
    """One group's rows stacked beyond round 1's 64-row tcgen05 limit: 64 rows x 2 heads (128 query
    rows, one M tile), the 4B shape with 64 live rows x 4 heads (256 rows, two M tiles; SURVEY §8d
    "R_h = 256"), and the CUDA-core prefix on the same layout."""
    lens = _lens(64, 1, grp_rows, rot=grp_rows + Hq)
    _check(lib, 64, 1, grp_rows, 255, Hq, Hkv, lens, impl, seed=grp_rows * 7 + Hq)


@pytest.mark.parametrize("qscale,exact", [(1.0, True), (4.0, False), (3.2, False)])
def test_split_attention_prefix_offset_paths(lib, monkeypatch, qscale, exact):
    """The tcgen05 prefix softmax takes the Cauchy-Schwarz bound B = ||q|| max_t ||k_t|| / sqrt(d)
    as its offset when every column's B <= 40 (exp(s - B) in [e^-80, 1]), else the exact column
    max; IS_EXACT_PREFIX_MAX forces the latter.  Both equal the fp64 oracle: qscale 1 (B ~ 14,
    bound path unless forced), 4 (B ~ 56: every CTA falls back), 3.2 (B straddles 40 across
    CTAs: mixed)."""
    if exact:
        monkeypatch.setenv("IS_EXACT_PREFIX_MAX", "1")
    for rows, groups, grp_rows in [(16, 1, 8), (64, 8, 8), (16, 1, 16)]:
        lens = _lens(rows, groups, grp_rows, rot=int(qscale * 10))
        _check(lib, rows, groups, grp_rows, 255, 16, 8, lens, 0, seed=int(qscale * 100) + rows, qscale=qscale)
