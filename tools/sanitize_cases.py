"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  usage: python tools/sanitize_cases.py CASE   (linalg, slots, encode, mgd3,
mgd4, mlp, dp, store)  -- each case ends by checking its result against the oracle so a run that
the sanitizer lets through is also a correct one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1702_06943_b200 import _native as N, codec, synth  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402

case = sys.argv[1]
O.build()


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def cfg2(nb):
    rp, c, v, counts = synth.cfg2_batches_csr(7, range(nb), 250, 784)
    br = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return rp, c, v, br


def oracle_sweep(rp, c, v, br, vv, uu):
    R, Os = [], []
    for b in range(len(br) - 1):
        lo, hi = rp[br[b]], rp[br[b + 1]]
        t = O.Tree.from_encoding(O.encode_csr(784, rp[br[b]:br[b + 1] + 1] - lo, c[lo:hi], v[lo:hi]))
        R.append(t.matvec(vv))
        Os.append(t.vecmat(uu[br[b]:br[b + 1]]))
    return np.concatenate(R), np.stack(Os)


if case in ("linalg", "slots", "encode"):
    nb = 3
    rp, c, v, br = cfg2(nb)
    arena = codec.compress_csr(784, rp, c, v, br)
    rng = np.random.default_rng(1)
    vv, uu = rng.standard_normal(784), rng.standard_normal(int(br[-1]))
    vd, ud = torch.from_numpy(vv).cuda(), torch.from_numpy(uu).cuda()
    wantR, wantO = oracle_sweep(rp, c, v, br, vv, uu)
    runs = []
    if case == "encode":
        got = arena.decode()
        assert got is not None
        runs.append(("block", arena.linalg(3, v=vd, u=ud, use_trees=False, use_levels=False)))
    elif case == "linalg":
        runs.append(("block", arena.linalg(3, v=vd, u=ud, use_trees=False, use_levels=False)))
        arena.build_trees()
        for k in (1, 2, 3):
            runs.append((f"trees{k}", arena.linalg(k, v=vd, u=ud, use_levels=False)))
        R32, O32 = arena.linalg32(3, v=vd.float(), u=ud.float())
        assert rel(R32.double().cpu(), wantR) < 1e-4 and rel(O32.double().cpu(), wantO) < 1e-4
    else:
        assert arena.build_levels()
        for k in (1, 2, 3):
            runs.append((f"slots{k}", arena.linalg(k, v=vd, u=ud)))
        for k in (1, 2, 3):  # the fp32 slot kernel (toc_linalg_levels32), fixed point and float atomics
            for scale in (1.0, None):
                u32 = ud.float() if scale else (ud * torch.pow(10.0, 16 * torch.rand_like(ud) - 8)).float()
                want_o = wantO if scale else oracle_sweep(rp, c, v, br, vv, u32.double().cpu().numpy())[1]
                R32, O32 = arena.linalg32(k, v=vd.float(), u=u32)
                if k & 1:
                    assert rel(R32.double().cpu(), wantR) < 1e-4
                if k & 2:
                    assert rel(O32.double().cpu(), want_o) < 1e-4
    for name, (R, Ox) in runs:
        if R is not None and name[-1] in "13k":
            assert rel(R.cpu(), wantR) < 1e-9, (name, rel(R.cpu(), wantR))
        if Ox is not None and name[-1] in "23k":
            assert rel(Ox.cpu(), wantO) < 1e-9, (name, rel(Ox.cpu(), wantO))
elif case in ("mgd3", "mgd4"):
    from paper_1702_06943_b200.training import DeviceBatches, GlmTrainer, shuffle_order

    if case == "mgd3":
        n, m, loss, lr = 1500, 68, "logistic", 0.1
        rp, c, v, y = synth.cfg3_dataset(n, seed=5)
        modes = ["images", "relay"]
    else:
        n, m, loss, lr = 1000, 47236, "hinge", 0.01
        rp, c, v, y = synth.cfg4_dataset(n)
        modes = ["parts", "relay"]
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(m, rp, c, v, check=False), labels=y)
    order = shuffle_order(n, 0)
    sh = LabeledDataset(features=ds.features.take_rows(order), labels=y[order])
    w_ref, _ = O.train_glm(rp, c, v, y, m, loss, 250, lr, 1, 0)
    for mode in modes:
        tr = GlmTrainer(DeviceBatches(sh, 250), loss, lr, mode=mode)
        assert tr.mode == mode, (tr.mode, mode)
        tr.epoch()
        got = tr.w.cpu().numpy()[:m]
        assert rel(got, w_ref) < 1e-9, (mode, rel(got, w_ref))
elif case == "mlp":
    from paper_1702_06943_b200.mlp import train_mlp

    rp, c, v, y = synth.cfg5_dataset(500)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v, check=False), labels=y)
    model, trace = train_mlp(ds, hidden=24, epochs=1)
    (w1r, b1r, w2r, b2r), _ = O.train_mlp(rp, c, v, y, 784, 24, 10, 250, 0.05, 1, 0)
    assert rel(model.w1, w1r) < 1e-6 and rel(model.w2, w2r) < 1e-6
elif case == "dp":
    from paper_1702_06943_b200.distributed import EmulatedDPEpochs

    rp, c, v, y = synth.cfg3_dataset(2 * 250 * 3, seed=9)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(68, rp, c, v), labels=y)
    run = EmulatedDPEpochs(ds, 250, 2, "logistic", 0.05)
    ws = run.epoch()
    w_ref, _ = O.train_glm(rp, c, v, y, 68, "logistic", 500, 0.05, 1, 0)
    assert rel(ws[0].cpu().numpy()[:68], w_ref) < 1e-9
else:
    raise SystemExit(f"unknown case {case}")
torch.cuda.synchronize()
print("case", case, "ok", os.path.basename(N.LIB_PATH))
