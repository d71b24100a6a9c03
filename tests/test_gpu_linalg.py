"""GPU parity: compressed A.v / v^T.A over device-resident TOC1 blocks vs the oracle.

Tolerance: 1e-9 relative in the reference's within_rel form (BASELINE.json north_star; the
reference's own bar, test_acceptance.py:139-203).  A.v is evaluated in a different summation
order than the reference (warp-parallel), so it is not required to be bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import max_rel_err, within_rel
from helpers import TOY_ROWS, TREE_ROWS, random_alphabet_rows

pytestmark = pytest.mark.gpu

REL = 1e-9


def _arena(blocks):
    from paper_1702_06943_b200.arena import BlockArena

    return BlockArena.from_bytes(blocks)


@pytest.fixture(params=["rebuild", "tree_cache", "levels"])
def tree_mode(request):
    return request.param


def _check_sweep(oracle, encs, v, seed=0, mode="rebuild"):
    import torch

    blocks = [oracle.serialize(e) for e in encs]
    arena = _arena(blocks)
    if mode == "tree_cache":
        arena.build_trees()
    if mode == "levels":
        # the slot cache takes every batch whose slots fit 15 bits; wider ones keep the other paths
        built = arena.build_levels()
        assert built or max(e.tree_length() for e in encs) > 32767
    trees = [oracle.Tree.from_encoding(e) for e in encs]
    n_total = sum(e.n_rows for e in encs)
    u = np.random.default_rng(seed).standard_normal(n_total)
    vd = torch.from_numpy(np.asarray(v, np.float64)).cuda()
    ud = torch.from_numpy(u).cuda()
    from paper_1702_06943_b200 import _native as N

    for kind in (N.TOC_MATVEC, N.TOC_VECMAT, N.TOC_MATVEC | N.TOC_VECMAT):
        R, O = arena.linalg(kind, v=vd if kind & 1 else None, u=ud if kind & 2 else None, use_levels=mode == "levels")
        torch.cuda.synchronize()
        base = 0
        for b, (e, t) in enumerate(zip(encs, trees)):
            if kind & N.TOC_MATVEC:
                want = t.matvec(v)
                got = R[base : base + e.n_rows].cpu().numpy()
                assert within_rel(got, want, REL), (kind, b, max_rel_err(got, want))
            if kind & N.TOC_VECMAT:
                want = t.vecmat(u[base : base + e.n_rows])
                got = O[b].cpu().numpy()
                assert within_rel(got, want, REL), (kind, b, max_rel_err(got, want))
            base += e.n_rows


def test_toy_known_answers(oracle):
    import torch

    enc = oracle.encode_rows(5, TOY_ROWS)
    arena = _arena([oracle.serialize(enc)])
    R = arena.matvec(torch.ones(5, dtype=torch.float64, device="cuda"))
    O = arena.vecmat(torch.ones(2, dtype=torch.float64, device="cuda"))
    assert R.cpu().tolist() == [15.0, 25.0]  # reference tests/test_kernels.py:55-62
    assert O[0].cpu().tolist() == [7.0, 9.0, 6.0, 8.0, 10.0]  # test_kernels.py:64-69


def test_tree_example(oracle, tree_mode):
    enc = oracle.encode_rows(5, TREE_ROWS)
    _check_sweep(oracle, [enc], np.arange(1.0, 6.0), mode=tree_mode)


def test_random_alphabet_many_blocks(oracle, tree_mode):
    rng = np.random.default_rng(7)
    encs = []
    n_cols = 12
    for i in range(60):
        rows = random_alphabet_rows(rng, int(rng.integers(0, 40)), n_cols, float(rng.uniform(0.05, 1.0)),
                                    16, integer_alphabet=bool(i % 2))
        encs.append(oracle.encode_rows(n_cols, rows))
    _check_sweep(oracle, encs, rng.standard_normal(n_cols), seed=1, mode=tree_mode)


def test_cfg1_batch(oracle, tree_mode):
    from paper_1702_06943_b200 import synth

    A = synth.cfg1_dense(0)
    enc = oracle.encode_csr(128, *synth.dense_to_csr(A))
    v, u = synth.cfg1_operands(0)
    _check_sweep(oracle, [enc], v, mode=tree_mode)


def test_cfg2_batches(oracle, tree_mode):
    from paper_1702_06943_b200 import synth

    encs = []
    for b in range(6):
        enc = oracle.encode_csr(784, *synth.dense_to_csr(synth.cfg2_batch_dense(0, b)))
        encs.append(enc)
    v, _ = synth.cfg2_operands(0, 6)
    _check_sweep(oracle, encs, v, seed=3, mode=tree_mode)


def test_levels_used_for_config2(oracle):
    """Config-2 batches take the level-cache kernel (the bench's headline path)."""
    from paper_1702_06943_b200 import synth

    encs = [oracle.encode_csr(784, *synth.dense_to_csr(synth.cfg2_batch_dense(0, b))) for b in range(4)]
    arena = _arena([oracle.serialize(e) for e in encs])
    assert arena.build_levels()
    assert arena.levels is not None and arena.levels_bytes > 0


def test_empty_and_zero_rows(oracle, tree_mode):
    encs = [oracle.encode_rows(4, []), oracle.encode_rows(3, [[(1, 2.0)], [], [(0, 4.0)]]),
            oracle.encode_rows(3, [[], []])]
    # n_cols differ from 4 -> keep one arena per n_cols
    _check_sweep(oracle, encs[1:], np.array([1.0, 1.0, 1.0]), mode=tree_mode)
    _check_sweep(oracle, encs[:1], np.ones(4), mode=tree_mode)


def test_long_record_streams(oracle, tree_mode):
    """Batches whose record stream (one 16-bit record per slot reference, toc_levels.cu) exceeds
    1024 x 32 records -- per-thread ranges of 40 records and more -- beside a short and an
    all-empty batch in the same launch, and empty rows between long ones."""
    from paper_1702_06943_b200 import synth

    rng = np.random.default_rng(17)
    big = synth.cfg2_batch_dense(0, 40, n_rows=280)  # ~34 k records, ~15.7 k slots: still the slot kernel
    big[5] = 0.0
    big[6] = 0.0
    big[-1] = 0.0
    encs = [oracle.encode_csr(784, *synth.dense_to_csr(big)),
            oracle.encode_csr(784, *synth.dense_to_csr(synth.cfg2_batch_dense(0, 42)[:7])),
            oracle.encode_csr(784, *synth.dense_to_csr(np.zeros((3, 784)))),
            oracle.encode_csr(784, *synth.dense_to_csr(synth.cfg2_batch_dense(0, 43)))]
    assert len(encs[0].codes) > 26000
    if tree_mode == "levels":
        arena = _arena([oracle.serialize(e) for e in encs])
        assert arena.build_levels(), "every batch here fits the slot cache"
    _check_sweep(oracle, encs, rng.standard_normal(784), seed=21, mode=tree_mode)


def test_wide_tree_global_tables(oracle, tree_mode):
    """A batch whose tree exceeds 65536 nodes (32-bit node ids) and shared memory (global
    table fallback): identical rows compress into long chains."""
    rng = np.random.default_rng(5)
    n_cols = 400
    base = random_alphabet_rows(rng, 30, n_cols, 0.9, 64)
    rows = [base[i % 30] if i % 3 else random_alphabet_rows(rng, 1, n_cols, 0.9, 64)[0] for i in range(600)]
    enc = oracle.encode_rows(n_cols, rows)
    assert enc.tree_length() > 65536
    _check_sweep(oracle, [enc], rng.standard_normal(n_cols), seed=9, mode=tree_mode)


def test_batch_sweep_public_api(oracle):
    """BatchSweep (host blocks in, host results out, chunked + overlapped) equals per-batch oracle."""
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.codec import compress_csr
    from paper_1702_06943_b200.kernels import BatchSweep

    nb = 13
    rp, c, v, counts = synth.cfg2_batches_csr(5, range(nb))
    br = np.concatenate([[0], np.cumsum(counts)])
    arena = compress_csr(784, rp, c, v, br)
    end = int(arena.block_off[-1] + arena.block_len[-1])
    host = arena.data[:end].cpu().numpy()
    sweep = BatchSweep.from_host_blocks(host, arena.block_off, arena.block_len, chunks=4)
    x, u = synth.cfg2_operands(5, nb)
    for _ in range(2):
        R, O = sweep.run(x, u)
    for b in range(nb):
        t = oracle.Tree.from_block(host[arena.block_off[b] : arena.block_off[b] + arena.block_len[b]].tobytes())
        assert within_rel(R[250 * b : 250 * (b + 1)], t.matvec(x), REL)
        assert within_rel(O[b], t.vecmat(u[250 * b : 250 * (b + 1)]), REL)
    assert sweep.h2d_bytes == end + 8 * 784 + 8 * 250 * nb
    # results are the caller's: a later run does not change them; out= fills the caller's buffers
    import torch

    R0, O0 = R.copy(), O.copy()
    sweep.run(-x, -u)
    assert np.array_equal(R, R0) and np.array_equal(O, O0)
    out = (torch.empty(250 * nb, dtype=torch.float64).pin_memory(), torch.empty((nb, 784), dtype=torch.float64).pin_memory())
    Ro, Oo = sweep.run(x, u, out=out)
    assert Ro is out[0] and np.array_equal(out[0].numpy(), R0) and np.array_equal(out[1].numpy(), O0)
    other = BatchSweep.from_host_blocks(host, arena.block_off, arena.block_len, chunks=3)  # its own events
    R2, O2 = other.run(x, u)
    assert np.array_equal(R2, R0) and np.array_equal(O2, O0)
    # pinned float64 operands are copied from in place (no staging); same results
    xp, up = torch.from_numpy(x).pin_memory(), torch.from_numpy(u).pin_memory()
    R3, O3 = sweep.run(xp, up)
    assert np.array_equal(R3, R0) and np.array_equal(O3, O0)
    with pytest.raises(ValueError):  # a wrong length is still refused (through the staging path)
        sweep.run(xp[:-1], up)
    # submit / finish: two sweeps over the same host blocks keep two steps in flight; each step's
    # results land in its own buffers and equal run()'s
    outs = [(torch.empty(250 * nb, dtype=torch.float64).pin_memory(),
             torch.empty((nb, 784), dtype=torch.float64).pin_memory()) for _ in range(2)]
    pair = [sweep, other]
    ops = [(xp, up), (torch.from_numpy(-x).pin_memory(), torch.from_numpy(-u).pin_memory())]
    pair[0].submit(*ops[0], out=outs[0])
    for i in range(1, 6):
        pair[i & 1].submit(*ops[i & 1], out=outs[i & 1])
        Rf, Of = pair[(i - 1) & 1].finish()
        sign = 1.0 if (i - 1) & 1 == 0 else -1.0
        assert Rf is outs[(i - 1) & 1][0] and np.array_equal(Rf.numpy(), sign * R0) and np.array_equal(Of.numpy(), sign * O0)
    pair[1].finish()
    assert np.array_equal(outs[1][0].numpy(), -R0) and np.array_equal(outs[1][1].numpy(), -O0)
    with pytest.raises(RuntimeError):
        sweep.finish()  # nothing submitted
    sweep.submit(xp, up)
    with pytest.raises(RuntimeError):
        sweep.submit(xp, up)  # one step per object in flight
    R4, O4 = sweep.finish()
    assert np.array_equal(R4, R0) and np.array_equal(O4, O0)


@pytest.mark.parametrize("kind", [1, 2, 3])
def test_fp32_variant_vs_oracle(oracle, kind):
    """The fp32 variant (toc_linalg32, fused walk for kind 3) within 1e-4 of the fp64 oracle -- the
    north_star's bar for it -- on config-2 batches, config 1 and a random alphabet with empty rows."""
    import torch

    from paper_1702_06943_b200 import synth

    cases = [[oracle.encode_csr(784, *synth.dense_to_csr(synth.cfg2_batch_dense(2, b))) for b in range(4)],
             [oracle.encode_csr(128, *synth.dense_to_csr(synth.cfg1_dense(0)))],
             [oracle.encode_rows(30, random_alphabet_rows(np.random.default_rng(8), 90, 30, 0.4) + [[]]),
              oracle.encode_rows(30, random_alphabet_rows(np.random.default_rng(9), 41, 30, 0.7))]]
    for encs in cases:
        m = encs[0].n_cols
        arena = _arena([oracle.serialize(e) for e in encs])
        rng = np.random.default_rng(kind)
        v = rng.standard_normal(m).astype(np.float32)
        u = rng.standard_normal(sum(e.n_rows for e in encs)).astype(np.float32)
        for slots in (False, True):  # over the tree cache (toc_linalg32), then over the slot cache (toc_linalg_levels32)
            if slots:
                assert arena.build_levels()
            R, O = arena.linalg32(kind, v=torch.from_numpy(v).cuda(), u=torch.from_numpy(u).cuda())
            base = 0
            for b, e in enumerate(encs):
                t = oracle.Tree.from_encoding(e)
                if kind & 1:
                    want = t.matvec(v.astype(np.float64))
                    got = R[base : base + e.n_rows].cpu().numpy().astype(np.float64)
                    assert within_rel(got, want, 1e-4), (slots, max_rel_err(got, want))
                if kind & 2:
                    want = t.vecmat(u[base : base + e.n_rows].astype(np.float64))
                    got = O[b].cpu().numpy().astype(np.float64)
                    assert within_rel(got, want, 1e-4), (slots, max_rel_err(got, want))
                base += e.n_rows


def test_linalg_pipelined_equals_linalg(oracle):
    """BlockArena.linalg_pipelined (host operands / results, sliced and overlapped) gives exactly
    the per-batch results of the one-launch call."""
    import torch

    from paper_1702_06943_b200 import _native as N, synth

    encs = [oracle.encode_csr(784, *synth.dense_to_csr(synth.cfg2_batch_dense(4, b))) for b in range(7)]
    arena = _arena([oracle.serialize(e) for e in encs])
    arena.build_trees()
    rng = np.random.default_rng(2)
    v = torch.from_numpy(rng.standard_normal(784)).pin_memory()
    u = torch.from_numpy(rng.standard_normal(arena.n_rows_total)).pin_memory()
    kind = N.TOC_MATVEC | N.TOC_VECMAT
    R0, O0 = arena.linalg(kind, v=v.cuda(), u=u.cuda())
    R = torch.empty(arena.n_rows_total, dtype=torch.float64).pin_memory()
    O = torch.empty((arena.n_blocks, 784), dtype=torch.float64).pin_memory()
    for chunks in (1, 3, 7):
        for _ in range(3):  # eager, then captured into a CUDA graph, then replayed
            R.zero_()
            O.zero_()
            arena.linalg_pipelined(kind, v, u, R, O, chunks=chunks)
            assert torch.equal(R, R0.cpu()) and torch.equal(O, O0.cpu())
    # the slot cache's kernel, two steps in flight on two sets of device buffers (new operands in
    # the same pinned tensors are picked up by the replayed graph)
    assert arena.build_levels()
    outs = [(torch.empty_like(R).pin_memory(), torch.empty_like(O).pin_memory()) for _ in range(2)]
    for rnd in range(2):
        if rnd == 1:  # new operands in the same pinned tensors (no step in flight while they change)
            v.mul_(-2.0)
            u.mul_(0.5)
        R0, O0 = arena.linalg(kind, v=v.cuda(), u=u.cuda())  # the slot kernel, one launch
        for it in range(5):
            s_ = it & 1
            arena.pipelined_wait(s_)
            if it >= 2:
                assert torch.equal(outs[s_][0], R0.cpu()) and torch.equal(outs[s_][1], O0.cpu())
            outs[s_][0].zero_()
            outs[s_][1].zero_()
            arena.linalg_pipelined(kind, v, u, outs[s_][0], outs[s_][1], chunks=4, slot=s_, wait=False)
        for s_ in (0, 1):
            arena.pipelined_wait(s_)
            assert torch.equal(outs[s_][0], R0.cpu()) and torch.equal(outs[s_][1], O0.cpu())



def _heavy_u(rng, n, kind):
    if kind == "outlier":  # one row weight ~1e7 among N(0,1) values (the rest keep |want| ~ 1)
        u = rng.standard_normal(n)
        u[int(rng.integers(0, n))] = 3.0e7
        return u
    return rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 8, n)  # N(0,1) * 10^U(-8, 8)


@pytest.mark.parametrize("u_kind", ["outlier", "heavy_tailed"])
def test_vecmat_heavy_tailed_u(oracle, tree_mode, u_kind):
    """v^T.A stays within the bar when the row weights span many orders of magnitude.  The
    fixed-point accumulation quantises every addend relative to the batch's sum |u|; batches where
    that could cost more than 2^-31 per output fall back to fp64 accumulation.  Checked in the
    reference's within_rel form AND pure-relative against each column's own magnitude:
    |got - want| <= 1e-9 |want| + 1e-13 S_c with S_c = sum_r |u_r a_rc| (the reference's own
    rounding scale)."""
    import torch

    from paper_1702_06943_b200 import _native as N
    from paper_1702_06943_b200 import synth

    dense = [synth.cfg2_batch_dense(11, b) for b in range(3)]
    encs = [oracle.encode_csr(784, *synth.dense_to_csr(A)) for A in dense]
    arena = _arena([oracle.serialize(e) for e in encs])
    if tree_mode == "tree_cache":
        arena.build_trees()
    if tree_mode == "levels":
        assert arena.build_levels()
    rng = np.random.default_rng(17)
    u = _heavy_u(rng, 750, u_kind)
    _, O = arena.linalg(N.TOC_VECMAT, u=torch.from_numpy(u).cuda(), use_levels=tree_mode == "levels")
    O = O.cpu().numpy()
    for b, (e, A) in enumerate(zip(encs, dense)):
        ub = u[250 * b : 250 * (b + 1)]
        want = oracle.Tree.from_encoding(e).vecmat(ub)
        scale = np.abs(ub) @ np.abs(A)
        assert within_rel(O[b], want, REL), max_rel_err(O[b], want)
        err = np.abs(O[b] - want)
        assert np.all(err <= 1e-9 * np.abs(want) + 1e-13 * scale), float(np.max(err / (np.abs(want) + scale)))


@pytest.mark.parametrize("u_kind", ["outlier", "heavy_tailed"])
def test_fp32_variant_heavy_tailed_u(oracle, u_kind):
    """The fp32 variant's 32-bit fixed point falls back to fp32 accumulation when it would be too
    coarse (within 1e-4 of the fp64 oracle, fused and alone)."""
    import torch

    from paper_1702_06943_b200 import synth

    dense = [synth.cfg2_batch_dense(12, b) for b in range(3)]
    encs = [oracle.encode_csr(784, *synth.dense_to_csr(A)) for A in dense]
    arena = _arena([oracle.serialize(e) for e in encs])
    rng = np.random.default_rng(18)
    u = _heavy_u(rng, 750, u_kind).astype(np.float32)
    v = rng.standard_normal(784).astype(np.float32)
    for slots in (False, True):  # the tree-cache kernel, then the slot-cache kernel
        if slots:
            assert arena.build_levels()
        for kind in (2, 3):
            _, O = arena.linalg32(kind, v=torch.from_numpy(v).cuda(), u=torch.from_numpy(u).cuda())
            for b, e in enumerate(encs):
                want = oracle.Tree.from_encoding(e).vecmat(u[250 * b : 250 * (b + 1)].astype(np.float64))
                got = O[b].cpu().numpy().astype(np.float64)
                assert within_rel(got, want, 1e-4), (slots, kind, max_rel_err(got, want))
