"""Modelled shared-memory wavefronts of the slot kernel's two stream phases (CPU only).

Builds the slot-cache entries of a few config-2 batches with the library's host builder
(toc_levels_build) and counts, per warp and step of the code stream, the wavefronts of
  * the v^T.A scatter: 32-bit atomics on the low limb word q of reference a, then of reference b
    (lanes whose record has one); the high limb (word q ^ 1) costs the same.  One wavefront per
    lane in the most loaded bank (same-word atomics serialise too);
  * the A.v row gathers: 64-bit loads of H[slot]; per half-warp one wavefront per distinct
    8-byte word in the most loaded of the 16 bank pairs.
The ideal is one wavefront per 32-bit warp access and two per 64-bit access.  Used to choose the
record placement (schedule_banks in csrc/toc_levels.cu) before spending GPU time.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def model(st_raw: np.ndarray, T: int, K: int, C: int):
    """st_raw: the entry's stream as stored (interleaved), u32[T*K].  Returns modelled wavefronts."""
    k = np.arange(K)
    pos = (k[None, :] // 8) * 8 * T + 8 * np.arange(T)[:, None] + (k[None, :] % 8)
    st = st_raw[pos]  # [T, K]
    qa = st & 0x7FFF
    qb = np.zeros_like(qa)  # one reference per record
    act = np.broadcast_to((np.arange(T)[:, None] * K) < C, (T, K))  # inactive threads skip the walk
    W = T // 32
    at_a = at_b = ga = gb = 0
    ideal_at_a = ideal_at_b = ideal_ga = ideal_gb = 0
    for w in range(W):
        sl = slice(w * 32, w * 32 + 32)
        if not act[sl].any():
            break
        A, B, M = qa[sl], qb[sl], act[sl]
        for s in range(K):
            m = M[:, s]
            a = A[m, s]
            if a.size:
                at_a += np.bincount(a & 31, minlength=32).max()
                ideal_at_a += 1
                for half in (slice(0, 16), slice(16, 32)):
                    ah = A[half, s][M[half, s]]
                    if ah.size:
                        wds = np.unique(ah >> 1)
                        ga += np.bincount(wds & 15, minlength=16).max()
                        ideal_ga += 1
            mb = m & (B[:, s] != 0)
            b = B[mb, s]
            if b.size:
                at_b += np.bincount(b & 31, minlength=32).max()
                ideal_at_b += 1
                for half in (slice(0, 16), slice(16, 32)):
                    hb = B[half, s]
                    hb = hb[M[half, s] & (hb != 0)]
                    if hb.size:
                        wds = np.unique(hb >> 1)
                        gb += np.bincount(wds & 15, minlength=16).max()
                        ideal_gb += 1
    return dict(atom=2 * (at_a + at_b), atom_ideal=2 * (ideal_at_a + ideal_at_b), gather=ga + gb,
                gather_ideal=ideal_ga + ideal_gb)


def model_inner(inner_raw: np.ndarray, nP: int):
    """Push (32-bit atomics on the low limb of each chain slot; the high limb costs the same) and
    inner H (64-bit gathers) over the inner records, 32 consecutive inner slots per warp."""
    par = inner_raw & 0xFFFF  # references (word index of the low limb)
    key = inner_raw >> 16
    nQ = len(inner_raw)
    q_inner = 2 * nP + 2
    at = ga = at_i = ga_i = 0
    for w0 in range(0, nQ, 32):
        lanes = np.arange(w0, min(w0 + 32, nQ))
        cur_key = key[lanes].copy()
        cur_par = par[lanes].copy()
        alive = np.ones(len(lanes), bool)
        while alive.any():
            k_ = cur_key[alive]
            at += np.bincount(k_ & 31, minlength=32).max()
            at_i += 1
            idx = np.nonzero(alive)[0]
            for half in (idx[idx < 16], idx[idx >= 16]):
                if half.size:
                    ga += np.bincount(np.unique(cur_key[half] >> 1) & 15, minlength=16).max()
                    ga_i += 1
            nxt = alive & (cur_par >= q_inner)
            y = (cur_par[nxt] >> 1) - nP - 1
            cur_key[nxt] = key[y]
            cur_par[nxt] = par[y]
            alive = nxt
        root = cur_par  # every lane's root pair (added after the loop, lanes converged)
        at += np.bincount(root & 31, minlength=32).max()
        at_i += 1
        for half in (root[:16], root[16:]):
            if half.size:
                ga += np.bincount(np.unique(half >> 1) & 15, minlength=16).max()
                ga_i += 1
    return dict(push=2 * at, push_ideal=2 * at_i, innerH=ga, innerH_ideal=ga_i)


def model_pairs(prs: np.ndarray, T: int):
    """Column-partials pass: thread t walks pair slots [1 + tM, 1 + tM + M); per iteration the value
    index gather (64-bit, by value ref) and the v gather (64-bit, by column) of each half-warp."""
    nP = len(prs)
    M = ((nP + T - 1) // T) | 1
    ref = (prs >> 16) & 0x7FFF
    col = prs & 0xFFFF
    gu = gv = ideal = 0
    for w0 in range(0, T, 32):
        for i in range(M):
            for h0 in (w0, w0 + 16):
                k = (np.arange(h0, h0 + 16) * M + i)
                k = k[k < nP]
                if not k.size:
                    continue
                ideal += 1
                gu += np.bincount(np.unique(ref[k]) & 15, minlength=16).max()
                gv += np.bincount(np.unique(col[k]) & 15, minlength=16).max()
    return dict(uniq=gu, vcol=gv, pairs_ideal=ideal)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=4)
    args = ap.parse_args()
    from oracle import oracle as O
    from paper_1702_06943_b200 import synth
    import test_levels_cpu as TL

    O.build()
    blocks = []
    for b in range(args.batches):
        rp, c, v = synth.dense_to_csr(synth.cfg2_batch_dense(0, b))
        blocks.append(O.serialize(O.encode_csr(784, rp, c, v)))
    t0 = time.time()
    rc, buf, eo = TL.build(blocks)
    dt = time.time() - t0
    assert rc == 0
    tot = {}
    for b in range(args.batches):
        o = int(eo[b])
        h = TL.entry(buf, o)
        st_raw = np.frombuffer(buf, np.uint16, h["T"] * h["K"], o + h["off_stream"]).astype(np.int64)
        r = model(st_raw, h["T"], h["K"], h["C"])
        r.update(model_pairs(np.frombuffer(buf, np.uint32, h["nP"], o + h["off_prs"]).astype(np.int64), h["T"]))
        r.update(model_inner(np.frombuffer(buf, np.uint32, h["nQ"], o + h["off_inner"]).astype(np.int64), h["nP"]))
        for k_, v_ in r.items():
            tot[k_] = tot.get(k_, 0) + v_
    n = args.batches
    print(f"build {dt / n * 1e3:.1f} ms per batch (2 threads)")
    print("per batch: " + "  ".join(f"{k_} {v_ / n:.0f}" for k_, v_ in tot.items()))


if __name__ == "__main__":
    main()
