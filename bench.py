#!/usr/bin/env python
"""Benchmark of the TOC hot path on B200 (BASELINE.json metric, config 2 = the matrix-op sweep).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over this GPU's shard of config 2: A.v AND v^T.A over 1024
compressed 250x784 float64 mini-batches (one fused launch reads each TOC1 block once for the
pair).  Batches shard across ranks with no collective (weak scaling); time is the max over ranks
of the device time (CUDA events) of the K timed steps; L2 (126 MB, larger than one shard's 87 MB
of blocks) is flushed by a 256 MiB write between steps, outside the events.

Prints ONE JSON line on rank 0 (contract in the task statement): value (rows/s, whole job),
roofline of the dominant kernel, cpu_baseline (the oracle port on this host's cores, rank 0 at
N=1, bounded sample), e2e (same metric through the public API with host buffers), clocks.
``--impl reference`` times the CPU oracle port (the reference is pure Python and cannot run on
the GPU box) on the same config and prints the same line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TOC A·v / vᵀ·A rows/s and MGD epoch seconds; % of HBM roofline, 1/2/4/8 GPU"
ROWS, COLS, BATCHES_PER_GPU, SEED = 250, 784, 1024, 20261020


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--batches-per-gpu", type=int, default=BATCHES_PER_GPU)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=20)
    p.add_argument("--no-mgd", action="store_true", help="skip the MGD epoch measurements (configs 3, 4, 5)")
    return p.parse_args()


# Exercise the N>1 MGD code paths (data-parallel trainers over NCCL) on one GPU: torchrun with one
# rank and BENCH_FORCE_DP=1.  A check of the multi-GPU path's mechanics, not a measurement mode.
FORCE_DP = os.environ.get("BENCH_FORCE_DP", "0") == "1"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def launch_ranks(args) -> None:
    """``--gpus N`` without a launcher: re-run this command under torchrun with N ranks (one per
    GPU, rendezvous on 127.0.0.1) and exit with its status.  Under a launcher, --gpus must equal
    WORLD_SIZE.  Never runs more ranks than visible GPUs: that fails loudly instead."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if args.gpus != world and not FORCE_DP:
            sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks")
        return
    if args.gpus <= 1:
        return
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, {have} visible")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region (NVML, 20 ms period)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def make_shard(rank: int, nb: int):
    """Config-2 batches [rank*nb, (rank+1)*nb) (seeded per batch) as concatenated CSR."""
    from paper_1702_06943_b200 import synth

    rp, c, v, counts = synth.cfg2_batches_csr(SEED, range(rank * nb, (rank + 1) * nb), ROWS, COLS)
    batch_row = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return rp, c, v, batch_row


def algorithmic_bytes(arena, kind: int) -> int:
    """TOC1 blocks read once, v read once, the outputs written,
    u read (v^T.A).  Per launch over the whole shard."""
    m = arena.n_cols
    n = arena.n_rows_total
    b = arena.block_bytes + 68 * arena.n_blocks  # blocks + their 68-byte index records
    if kind & 1:
        b += 8 * m + 8 * n
    if kind & 2:
        b += 8 * n + 8 * m * arena.n_blocks
    return b


def time_kernel(torch, fn, steps: int, warmup: int, flush):
    """Per-step device time (CUDA events on the launching stream) with an L2 flush between steps,
    outside the events.  Returns the list of step durations in ms."""
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        flush.fill_(1)
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(s)
        fn()
        ev[i][1].record(s)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def cpu_reference(arena_bytes_h, block_off, block_len, v, u, row_base, budget_s: float, steps: int,
                  warmup: int, oracle_mod):
    """The oracle port timed on this host (trees built outside the timed region, like the
    reference's own bench-kernels, cli.py:316-317).  Returns (rows/s, sample description, cores)."""
    O = oracle_mod
    O.build()
    nb = len(block_off)
    trees = [O.Tree.from_block(bytes(arena_bytes_h[block_off[b] : block_off[b] + block_len[b]])) for b in range(nb)]
    threads = O.max_threads()
    # calibrate: one sweep over min(64, nb) batches
    k = min(64, nb)
    t0 = time.perf_counter()
    O.sweep(trees[:k], row_base[:k], v, u, 2, threads)
    per_batch = max((time.perf_counter() - t0) / k, 1e-7)
    sample = int(max(1, min(nb, budget_s / max(steps + warmup, 1) / per_batch)))
    sel = trees[:sample]
    rb = row_base[:sample]
    for _ in range(warmup):
        O.sweep(sel, rb, v, u, 2, threads)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.sweep(sel, rb, v, u, 2, threads)
    dt = time.perf_counter() - t0
    rows = sample * ROWS * steps
    desc = (f"oracle port (C, OpenMP {threads} threads) A.v+v^T.A over the first {sample} of {nb} config-2 "
            f"batches x {steps} steps, trees prebuilt")
    return rows / dt, desc, threads, dt, trees


def _rel_err(got, want, pure: bool = False) -> float:
    """max |got - want| / max(1, |want|) (the reference's within_rel form), or relative to |want|
    itself with a 1e-12 x max|want| floor for exact zeros (pure)."""
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    if got.size == 0:
        return 0.0
    den = np.abs(want) + 1e-12 * np.max(np.abs(want)) + 1e-300 if pure else np.maximum(1.0, np.abs(want))
    return float(np.max(np.abs(got - want) / den))


def sweep_parity(O, trees, row_base, v, u, outputs):
    """Every batch's A.v and v^T.A from each timed mode against the oracle port's sweep over the
    same TOC1 blocks (bar 1e-9 for the f64 modes, 1e-4 for the fp32 variant)."""
    want_r, want_o = O.sweep(trees, row_base, v, u, 2, O.max_threads())
    out = {"batches": len(trees), "rows": int(len(want_r))}
    ok = True
    for name, (r, o) in outputs.items():
        bar = 1e-4 if name == "fp32_variant" else 1e-9
        e = {"matvec_max_rel": _rel_err(r, want_r), "vecmat_max_rel": _rel_err(o, want_o), "bar": bar}
        e["ok"] = e["matvec_max_rel"] <= bar and e["vecmat_max_rel"] <= bar
        ok &= e["ok"]
        out[name] = e
    out["ok"] = bool(ok)
    return out


def glm_parity(rp, c, v, y, m, loss, lr, epochs, batch, risks, weights):
    """The full-size MGD run against the oracle port's train (reference training.py:336-361) at
    the same global batch size: risk per epoch and final weights within 1e-6 relative (weights
    relative to each weight itself, not max(1, |w|))."""
    from oracle import oracle as O

    O.build()
    t0 = time.perf_counter()
    w_ref, risks_ref = O.train_glm(rp, c, v, y, m, loss, batch, lr, epochs, 0)
    e = {"global_batch": batch, "risk_max_rel": _rel_err(risks, risks_ref, pure=True),
         "weights_max_rel": _rel_err(weights, w_ref, pure=True), "bar": 1e-6,
         "nonzero_weights": int(np.count_nonzero(w_ref)), "oracle_seconds": time.perf_counter() - t0}
    e["ok"] = e["risk_max_rel"] <= 1e-6 and e["weights_max_rel"] <= 1e-6
    return e


def mlp_parity(steps: int = 40):
    """Config 5 at hidden = 200 over `steps` steps (250 * steps rows, one epoch) against the oracle's
    restatement (the reference has no such model: its first-layer matmat_right / matmat_left are
    the pinned parts)."""
    from oracle import oracle as O
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    O.build()
    rp, c, v, y = synth.cfg5_dataset(250 * steps)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v, check=False), labels=y)
    model, trace = train_mlp(ds, hidden=200, classes=10, batch_size=250, learning_rate=0.05, epochs=1, seed=0)
    (w1, b1, w2, b2), risks = O.train_mlp(rp, c, v, y, 784, 200, 10, 250, 0.05, 1, 0)
    e = {"steps": steps, "hidden": 200, "risk_max_rel": _rel_err(trace.risks, risks, pure=True),
         "params_max_rel": max(_rel_err(g, w, pure=True) for g, w in
                               ((model.w1, w1), (model.b1, b1), (model.w2, w2), (model.b2, b2))), "bar": 1e-6}
    e["ok"] = e["risk_max_rel"] <= 1e-6 and e["params_max_rel"] <= 1e-6
    return e


def memory_line(toc1: int, cache: int, nnz: int, rows: int, cols: int, what: str) -> dict:
    """Bytes resident for the run against the uncompressed forms of the same rows (the reference's
    own accounting, reports.py:38-55: CSR = 12 B per entry + 4 B per row pointer)."""
    csr = 12 * nnz + 4 * (rows + 1)
    dense = 8 * rows * cols
    return {"toc1_bytes": int(toc1), "cache_bytes": int(cache), "cache": what, "csr_bytes": int(csr),
            "dense_bytes": int(dense), "cache_over_toc1": cache / max(toc1, 1), "cache_over_csr": cache / csr,
            "cache_over_dense": cache / max(dense, 1), "toc1_over_csr": toc1 / csr}


_RESULT = None  # the real stdout: only the result line goes there


def claim_stdout():
    """Send everything written to fd 1 (library banners such as NCCL's, warnings) to stderr, and
    keep the original stdout for the one JSON result line the driver parses."""
    global _RESULT
    if _RESULT is None:
        sys.stdout.flush()
        _RESULT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)
    return _RESULT


def smem_pipe_line(wavefronts, ms_per_step: float, clocks):
    """The kernel's shared-memory pipe fraction: shared wavefronts per launch (ncu, profiles/traffic.json)
    over what the 148 SMs' pipes (one 128-byte wavefront per SM per cycle) serve in the measured step
    at the sampled SM clock.  None without a capture."""
    if not wavefronts or not clocks or not clocks.get("sm_mhz"):
        return None
    cycles = ms_per_step / 1e3 * clocks["sm_mhz"] * 1e6
    return {"wavefronts_per_launch": wavefronts, "sm_cycles_per_launch": cycles, "sms": 148,
            "frac": wavefronts / (148 * cycles), "unit": "wavefronts per SM-cycle (peak 1)"}


def emit(line: dict) -> None:
    print(json.dumps(line), file=claim_stdout(), flush=True)


def main():
    args = parse()
    launch_ranks(args)
    claim_stdout()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch

    from paper_1702_06943_b200 import _native as N
    from paper_1702_06943_b200.codec import compress_csr

    torch.cuda.set_device(local)
    if world > 1 or FORCE_DP:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nb = args.batches_per_gpu
    t0 = time.perf_counter()
    rp, c, vals, batch_row = make_shard(rank, nb)
    t_gen = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    arena = compress_csr(COLS, rp, c, vals, batch_row)
    torch.cuda.synchronize()
    t_enc = time.perf_counter() - t0
    # encoder throughput (a second run, device time by CUDA events: the CSR upload, encode,
    # value index, widths and packing of every batch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    compress_csr(COLS, rp, c, vals, batch_row)
    e1.record()
    e1.synchronize()
    enc_ms = e0.elapsed_time(e1)
    rng = np.random.default_rng(np.random.SeedSequence([SEED, 7, rank]))
    v_h = rng.standard_normal(COLS)
    u_h = rng.standard_normal(arena.n_rows_total)
    v = torch.from_numpy(v_h).cuda()
    u = torch.from_numpy(u_h).cuda()
    kind = N.TOC_MATVEC | N.TOC_VECMAT
    R = torch.empty(arena.n_rows_total, dtype=torch.float64, device="cuda")
    O = torch.empty((arena.n_blocks, COLS), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    # per-batch caches (built once, outside the timed region -- like the reference's own
    # bench-kernels, which builds trees before timing, cli.py:316-317): the slot cache the headline
    # launch reads (toc_levels.cu) and the tree cache of the chain-walk kernel (reported beside it)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    arena.build_trees()
    torch.cuda.synchronize()
    t_trees = time.perf_counter() - t0
    t0 = time.perf_counter()
    slots = arena.build_levels()
    torch.cuda.synchronize()
    t_slots = time.perf_counter() - t0

    def step():  # the slot cache when it fits (config 2: always), else the tree cache
        arena.linalg(kind, v=v, u=u, R=R, O=O)

    sampler = ClockSampler(local)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with sampler:
        times = time_kernel(torch, step, args.steps, args.warmup, flush)
    total_ms = float(np.sum(times))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    rows_per_step = arena.n_rows_total  # per rank
    value = world * rows_per_step * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps
    outputs = {"headline": (R.cpu().numpy(), O.cpu().numpy())}  # checked against the oracle below

    # separate A.v-only and v^T.A-only launches (same protocol) for the per-op rows/s
    nsub = max(args.steps // 4, 10)
    mv_t = time_kernel(torch, lambda: arena.linalg(N.TOC_MATVEC, v=v, R=R), nsub, 3, flush)
    vm_t = time_kernel(torch, lambda: arena.linalg(N.TOC_VECMAT, u=u, O=O), nsub, 3, flush)
    outputs["separate"] = (R.cpu().numpy(), O.cpu().numpy())
    # block-only mode: the tree is rebuilt from the TOC1 codes inside every launch
    bo_t = time_kernel(torch, lambda: arena.linalg(kind, v=v, u=u, R=R, O=O, use_trees=False, use_levels=False),
                       nsub, 3, flush)
    outputs["block_only"] = (R.cpu().numpy(), O.cpu().numpy())
    # the chain-walk kernel over the tree cache (toc_linalg.cu), measured beside the headline
    tc_t = time_kernel(torch, lambda: arena.linalg(kind, v=v, u=u, R=R, O=O, use_levels=False), nsub, 3, flush)
    outputs["tree_cache"] = (R.cpu().numpy(), O.cpu().numpy())
    # the fp32 variant (north_star: 1e-4 bar): same batches, fused single walk for both products
    v32, u32 = v.float(), u.float()
    R32 = torch.empty_like(R, dtype=torch.float32)
    O32 = torch.empty_like(O, dtype=torch.float32)
    f32_t = time_kernel(torch, lambda: arena.linalg32(kind, v=v32, u=u32, R=R32, O=O32), nsub, 3, flush)
    outputs["fp32_variant"] = (R32.double().cpu().numpy(), O32.double().cpu().numpy())

    peak, peak_src = measured_peaks()
    alg = algorithmic_bytes(arena, kind)
    achieved = alg / (ms_per_step / 1e3) / 1e9
    traffic = bo_traffic = traffic_src = smem_wf = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):  # DRAM bytes per launch from the last ncu --set full capture (dated there)
        tj = json.load(open(tpath))
        traffic = tj.get("levels_kernel_both")  # the mode `value` is measured in (slot cache)
        bo_traffic = tj.get("linalg_kernel_both")
        traffic_src = {k: tj[k] for k in ("captured", "source", "kernel_build") if k in tj}
        smem_wf = tj.get("levels_kernel_both_smem_wavefronts")

    # ---- e2e: public API call with host buffers (pinned), copies inside the timed region ----
    e2e = run_e2e(torch, arena, v_h, u_h, args.e2e_steps, world)
    e2e_resident = run_e2e_resident(torch, arena, v_h, u_h, args.e2e_steps, world)

    cpu = None
    parity = {}
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as Omod

        data_h = arena.data.cpu().numpy()
        rps, desc, cores, dt, trees = cpu_reference(data_h, arena.block_off, arena.block_len, v_h, u_h,
                                                    arena.row_base, 12.0, 5, 1, Omod)
        cpu = {"value": rps, "unit": "rows/s", "cores": cores, "kind": "port", "sample": desc}
        parity["config2_sweep"] = sweep_parity(Omod, trees, arena.row_base, v_h, u_h, outputs)

    mgd = {}
    if not args.no_mgd:
        cs = rank == 0 and world == 1 and not args.no_cpu_baseline
        chk = rank == 0 and not args.no_cpu_baseline
        mgd["config3_logistic"] = run_mgd(3, rank, world, cpu_sample=cs, parity=parity if chk else None)
        mgd["config4_hinge"] = run_mgd(4, rank, world, cpu_sample=cs, parity=parity if chk else None)
        mgd["config5_mlp"] = run_mgd(5, rank, world, cpu_sample=cs)
        if chk and world == 1:
            parity["config5_40_steps"] = mlp_parity()
    if parity:
        parity["all_ok"] = all(p.get("ok", False) for p in parity.values() if isinstance(p, dict))

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "rows/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (config-2 generator, seeded; DESIGN.md)",
            "config": {
                "workload": f"config 2 sweep: {nb} TOC-compressed 250x784 f64 mini-batches per GPU; one step = "
                            "A.v and v^T.A over every batch in one fused launch",
                "batches_per_gpu": nb, "rows_per_batch": ROWS, "n_cols": COLS,
                "parallelism": f"batch-sharded x{world} (no collective)",
                "l2": "flushed between steps (256 MiB write outside the timed events)",
                "toc_block_bytes_per_gpu": arena.block_bytes,
                "csr_bytes_per_gpu": int(len(c) * 12 + (len(rp)) * 8),
                "encode_seconds": t_enc, "generate_seconds": t_gen,
            },
            "encode": {"ms": enc_ms, "rows_per_s": world * arena.n_rows_total / (enc_ms / 1e3),
                       "csr_in_bytes": int(len(c) * 12 + len(rp) * 8), "toc1_out_bytes": arena.block_bytes,
                       "csr_in_gbs": (len(c) * 12 + len(rp) * 8) / (enc_ms / 1e3) / 1e9,
                       "note": "codec.compress_csr device time (CUDA events), H2D of the CSR inputs included; "
                               "one CTA per batch, hash tables in global memory (latency-bound, DESIGN.md 4.2)"},
            "memory": memory_line(arena.block_bytes, arena.levels_bytes if slots else arena.tree_bytes, len(c),
                                  len(rp) - 1, COLS, "slot cache (read by every launch)" if slots
                                  else "tree cache (read by every launch)"),
            "parity": parity or None,
            "matvec_rows_per_s": world * rows_per_step / (np.mean(mv_t) / 1e3),
            "vecmat_rows_per_s": world * rows_per_step / (np.mean(vm_t) / 1e3),
            "slot_cache": {"used_for_value": bool(slots), "bytes_per_gpu": arena.levels_bytes if slots else None,
                           "build_seconds": t_slots,
                           "note": "toc_levels.cu, per-batch entry built once on the host (the reference caches "
                                   "C' too, kernels.py:68-77): value index, row offsets, column-sorted pair slots, "
                                   "inner-node (parent, key) records, the code stream as slot references cut into "
                                   "equal per-thread ranges (bank-aware placement); the launch reads only this"},
            "tree_cache": {"used_for_value": not slots, "bytes_per_gpu": arena.tree_bytes, "build_seconds": t_trees,
                           "ms_per_step": float(np.mean(tc_t)),
                           "rows_per_s": world * rows_per_step / (np.mean(tc_t) / 1e3),
                           "roofline_frac": alg / (np.mean(tc_t) / 1e3) / 1e9 / peak,
                           "note": "toc_linalg.cu chain walk over the device tree cache (decode-tree prefix plus "
                                   "unpacked and column-sorted pair records) and the TOC1 value index; round-1 "
                                   "headline, kept as the path for batches the slot cache does not fit"},
            "block_only": {"ms_per_step": float(np.mean(bo_t)),
                           "rows_per_s": world * rows_per_step / (np.mean(bo_t) / 1e3),
                           "roofline_frac": alg / (np.mean(bo_t) / 1e3) / 1e9 / peak, "traffic": bo_traffic,
                           "note": "tree rebuilt from the TOC1 codes inside every launch; reads only the block"},
            "fp32_variant": {"ms_per_step": float(np.mean(f32_t)),
                             "rows_per_s": world * rows_per_step / (np.mean(f32_t) / 1e3),
                             "roofline_frac": alg / (np.mean(f32_t) / 1e3) / 1e9 / peak, "dtype": "f32",
                             "note": "toc_linalg_levels32 over the slot cache (toc_linalg32 over the tree cache when "
                                     "there is none): fp32 operands and H, 32-bit fixed-point v^T.A (one atomic per "
                                     "record); 1e-4 of the fp64 oracle (not the headline: the reference is f64)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic if slots else None, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": alg,
                         "kernel": "toc::levels_kernel<3> (A.v + v^T.A, slot cache)" if slots
                         else "toc::linalg_kernel (A.v + v^T.A, tree cache)"},
            "smem_pipe": smem_pipe_line(smem_wf if slots else None, ms_per_step, sampler.summary()),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_resident": e2e_resident,
            "gpu_launches": args.steps,
            "clocks": sampler.summary(),
            "mgd": mgd,
        }
        emit(line)
    if world > 1 or FORCE_DP:
        torch.distributed.destroy_process_group()


def run_mgd(cfg: int, rank: int, world: int, cpu_sample: bool, parity=None):
    """MGD epoch seconds at the config's full size (BASELINE.json configs[2] / [3] / [4]).  N=1: one
    launch per epoch (GLMs: a thread-block cluster over cached step images when they fit shared
    memory, else the relay; config 5: per-step first-layer matmat kernels over the node-record
    cache plus torch for the dense tail); N>1: synchronous data parallel with NCCL (per-replica
    batch 250, global 250*N).  Device time (CUDA events), max over ranks.  One-time cache builds
    (the reference's once-only cached trees) are reported beside the epochs, not inside them."""
    import torch

    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.training import DeviceBatches, GlmTrainer, TrainConfig, shuffle_once

    if cfg == 5:
        return run_mlp(rank, world, cpu_sample)
    if cfg == 3:
        rp, c, v, y = synth.cfg3_dataset()
        m, loss, lr, epochs = 68, "logistic", 0.1, 10
    else:
        rp, c, v, y = synth.cfg4_dataset()
        m, loss, lr, epochs = 47_236, "hinge", 0.01, 5
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(m, rp, c, v, check=False), labels=y)
    out = {"rows": len(y), "n_cols": m, "loss": loss, "batch_size": 250, "lr": lr, "epochs": epochs}
    if world == 1 and not FORCE_DP:
        batches = DeviceBatches(shuffle_once(ds, 0), 250)
        tr = GlmTrainer(batches, loss, lr)
        secs, risks = [], []
        for _ in range(epochs):
            secs.append(tr.epoch())
            risks.append(tr.risk())
        modes = {"images": f"one launch per epoch: a {tr.cluster}-CTA thread-block cluster over cached step images "
                           "(built once per run, like the reference's cached trees)",
                 "parts": f"one launch per epoch: a {tr.cluster}-CTA cluster over per-CTA part images (built once per "
                          "run), weights and an exact fixed-point gradient in global memory",
                 "relay": "one cooperative relay launch per epoch (tables rebuilt per step)"}
        # HBM roofline of the epoch: each step reads its TOC1 block and labels once
        ep_bytes = batches.arena.block_bytes + 8 * len(y)
        peak, _ = measured_peaks()
        out["roofline"] = {"bound": "hbm (latency-bound dependency chain in practice)",
                           "algorithmic_bytes_per_epoch": int(ep_bytes),
                           "frac": ep_bytes / min(secs) / 1e9 / peak, "peak_gbs": peak,
                           "us_per_step": min(secs) / batches.arena.n_blocks * 1e6}
        out.update({"steps_per_epoch": int(batches.arena.n_blocks), "epoch_seconds": secs, "risk_per_epoch": risks,
                    "mode": modes[tr.mode], "image_build_seconds": tr.image_build_seconds,
                    "image_bytes": int(tr.image_off[-1]) if tr.mode in ("images", "parts") else 0})
        out["memory"] = memory_line(batches.arena.block_bytes, out["image_bytes"], len(c), len(y), m,
                                    f"{tr.mode} step images (read by every epoch)")
        if parity is not None:
            parity[f"config{cfg}_{loss}"] = glm_parity(rp, c, v, y, m, loss, lr, epochs, 250, risks, tr.weights())
        if cpu_sample:
            out["cpu_port"] = cpu_mgd_sample(rp, c, v, y, m, loss, lr, batches.arena.n_blocks,
                                             sample_batches=400 if cfg == 3 else 100)
    else:
        from paper_1702_06943_b200.distributed import train_data_parallel

        model, trace = train_data_parallel(ds, TrainConfig(loss, 250, lr, epochs), world, rank)
        if parity is not None:  # the data-parallel run is the reference's at the global batch 250 N
            parity[f"config{cfg}_{loss}"] = glm_parity(rp, c, v, y, m, loss, lr, epochs, 250 * world, trace.risks,
                                                       model.weights)
        out.update({"steps_per_epoch": -(-len(y) // (250 * world)), "epoch_seconds": trace.seconds,
                    "risk_per_epoch": trace.risks,
                    "mode": f"data parallel x{world}: " + (
                        "gradient exchange fused into the cluster epoch kernel over NVLink peer memory, one launch "
                        "per epoch" if getattr(trace, "mode", "") == "fused" else
                        "per step cluster gradient -> NCCL all-reduce -> update, one CUDA graph per epoch")})
    return out


def run_mlp(rank: int, world: int, cpu_sample: bool):
    """Config 5: 784-200-10 ReLU softmax-CE MLP, 1,000,000 rows, batch 250, lr 0.05, 5 epochs (N>1:
    synchronous data parallelism, global batch 250 N)."""
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    n, epochs = 1_000_000, 5
    out = {"rows": n, "n_cols": 784, "model": "784-200-10 ReLU softmax-CE f64", "batch_size": 250, "lr": 0.05,
           "epochs": epochs}
    rp, c, v, y = synth.cfg5_dataset(n)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v, check=False), labels=y)
    if world > 1 or FORCE_DP:
        from paper_1702_06943_b200.distributed import train_mlp_data_parallel

        _, trace = train_mlp_data_parallel(ds, world, rank, epochs=epochs)
        out.update({"steps_per_epoch": -(-n // (250 * world)), "epoch_seconds": trace.seconds,
                    "risk_per_epoch": trace.risks,
                    "mode": f"data parallel x{world}: per step toc_mlp_step_grad (native step kernels, gradient "
                            "only) -> NCCL all-reduce of the flat gradient -> update; one CUDA graph per epoch"})
        return out
    t0 = time.perf_counter()
    _, trace = train_mlp(ds, epochs=epochs)
    out.update({"steps_per_epoch": n // 250, "epoch_seconds": trace.seconds, "risk_per_epoch": trace.risks,
                "wall_seconds_incl_compress_and_cache": time.perf_counter() - t0,
                "memory": getattr(trace, "memory", None),
                "mode": "native epoch (toc_mlp_epoch, one CUDA graph): per step the batch decoded from its TOC1 "
                        "code stream and its step-cache entry (4-byte node records) into an L2-resident tile "
                        "buffer, A.W1 and A^T.delta on the fp64 tensor cores (DMMA), softmax-CE tail and parameter "
                        "updates in CUDA kernels"})
    if cpu_sample:
        out["cpu_port"] = cpu_mlp_sample(rp, c, v, y, n // 250)
    return out


def cpu_mlp_sample(rp, c, v, y, steps_full: int, sample_batches: int = 10):
    """The oracle's config-5 step (C matmat_right / matmat_left + numpy dense tail) on the first
    sample_batches batches, scaled to a full epoch.  Single thread."""
    from oracle import oracle as O

    O.build()
    k = 250 * sample_batches
    srp = rp[: k + 1]
    t0 = time.perf_counter()
    O.train_mlp(srp, c[: srp[-1]], v[: srp[-1]], y[:k], 784, 200, 10, 250, 0.05, 1, 0)
    dt = time.perf_counter() - t0
    return {"epoch_seconds_est": dt * steps_full / sample_batches,
            "sample": f"{sample_batches} of {steps_full} steps (incl. their tree builds), 1 thread", "kind": "port"}


def cpu_mgd_sample(rp, c, v, y, m, loss, lr, steps_full: int, sample_batches: int = 400):
    """The oracle port's MGD epoch time on a bounded sample (first sample_batches batches of the
    shuffled order, trees built outside the timing like the reference's own), scaled to a full
    epoch.  Single thread: MGD steps are sequential."""
    from oracle import oracle as O

    O.build()
    order = O.shuffle_order(len(y), 0)[: 250 * sample_batches]
    lens = np.diff(rp)[order]
    srp = np.concatenate([[0], np.cumsum(lens)])
    g = np.concatenate([np.arange(rp[i], rp[i + 1]) for i in order])
    trees, bases = O.make_batch_trees(srp, c[g], v[g], m, np.arange(len(order)), 250)
    ys = np.ascontiguousarray(y[order], np.float64)
    import ctypes as C

    handles = (C.c_void_p * len(trees))(*[t._h for t in trees])
    w = np.zeros(m)
    t0 = time.perf_counter()
    O.lib().or_glm_epoch(len(trees), handles, O._ptr(bases), O._ptr(ys), O._ptr(w), O.LOSS_CODE[loss], float(lr))
    dt = time.perf_counter() - t0
    return {"epoch_seconds_est": dt * steps_full / len(trees), "sample": f"{len(trees)} of {steps_full} steps, 1 thread",
            "kind": "port"}


def _wall_max(torch, dt: float, world: int) -> float:
    """Slowest rank's wall time (every rank runs its own shard concurrently)."""
    if world == 1:
        return dt
    t = torch.tensor([dt], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def _wall_start(torch, world: int) -> float:
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    return time.perf_counter()


def run_e2e(torch, arena, v_h, u_h, steps: int, world: int = 1):
    """Same metric through the public API: host TOC1 bytes + host v/u in pinned memory -> device
    (H2D inside the timed region) -> validate/index -> fused A.v + v^T.A -> host R/O (D2H)."""
    from paper_1702_06943_b200.kernels import BatchSweep

    blocks_h = arena.data[: int(arena.block_off[-1] + arena.block_len[-1])].cpu().numpy()
    # two sweeps over the same host blocks, submitted alternately (two steps in flight): while one
    # step's last chunks are validated, swept and downloaded, the next step's upload is under way
    sweeps = [BatchSweep.from_host_blocks(blocks_h, arena.block_off, arena.block_len) for _ in range(2)]
    sweep = sweeps[0]
    outs = [(torch.empty(sweep.n_rows, dtype=torch.float64).pin_memory(),  # the caller's pinned result buffers
             torch.empty((sweep.n_blocks, sweep.n_cols), dtype=torch.float64).pin_memory()) for _ in range(2)]
    vh, uh = torch.from_numpy(v_h).pin_memory(), torch.from_numpy(u_h).pin_memory()  # pinned operands
    for _ in range(2):
        sweep.run(vh, uh, out=outs[0])
        sweeps[1].run(vh, uh, out=outs[1])
    # one step at a time (run = submit + finish)
    t0 = _wall_start(torch, world)
    for _ in range(steps):
        sweep.run(vh, uh, out=outs[0])
    dt_serial = _wall_max(torch, time.perf_counter() - t0, world)
    # two steps in flight: every step still uploads its blocks and operands from pinned host memory
    # and downloads its R / O into the caller's pinned buffers inside the timed region
    t0 = _wall_start(torch, world)
    sweeps[0].submit(vh, uh, out=outs[0])
    for i in range(1, steps):
        sweeps[i & 1].submit(vh, uh, out=outs[i & 1])
        sweeps[(i - 1) & 1].finish()
    sweeps[(steps - 1) & 1].finish()
    dt = _wall_max(torch, time.perf_counter() - t0, world)
    same = bool(torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]))
    link = h2d_link_gbs(torch, sweep.h2d_bytes)
    achieved = sweep.h2d_bytes * steps / dt / 1e9
    return {"value": world * sweep.n_rows * steps / dt, "unit": "rows/s", "h2d_bytes_per_step": sweep.h2d_bytes,
            "d2h_bytes_per_step": sweep.d2h_bytes,
            "api": "paper_1702_06943_b200.kernels.BatchSweep.submit(v, u, out=(R, O)) / finish(): pinned host "
                   "blocks, v and u in, results into the caller's pinned buffers; two sweeps over the same host "
                   "blocks alternate, so two steps are in flight",
            "serial_value": world * sweep.n_rows * steps / dt_serial,
            "serial_api": "BatchSweep.run(v, u, out=(R, O)) = submit + finish, one step at a time",
            "both_sweeps_bit_identical": same,
            "h2d_gbs": achieved, "h2d_link_gbs": link, "link_frac": achieved / link if link else None,
            "link_note": "h2d_link_gbs: one pinned host->device copy of the same byte count, best of 5 "
                         "(CUDA events); the streamed TOC1 upload bounds this e2e number"}


def h2d_link_gbs(torch, nbytes: int) -> float:
    """Host->device bandwidth of this box's link for one pinned copy of `nbytes`."""
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = float("inf")
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del src, dst
    return nbytes / best / 1e9


def run_e2e_resident(torch, arena, v_h, u_h, steps: int, world: int = 1):
    """The same metric with the compressed arena resident in HBM (built once, like the reference's
    own bench-kernels keeps its CompressedMatrix objects, cli.py:299-334): per step v and u go
    host -> device from pinned memory, the fused launch runs, R and O come back to pinned host
    memory; wall clock around the whole step."""
    from paper_1702_06943_b200 import _native as N

    kind = N.TOC_MATVEC | N.TOC_VECMAT
    vh = torch.from_numpy(v_h).pin_memory()
    uh = torch.from_numpy(u_h).pin_memory()
    Rh = torch.empty(arena.n_rows_total, dtype=torch.float64).pin_memory()
    Oh = torch.empty((arena.n_blocks, arena.n_cols), dtype=torch.float64).pin_memory()

    def step():  # the public API: pinned host operands in, pinned host results out, pipelined
        arena.linalg_pipelined(kind, vh, uh, Rh, Oh, chunks=4)

    for _ in range(3):
        step()
    t0 = _wall_start(torch, world)
    for _ in range(steps):
        step()
    dt_serial = _wall_max(torch, time.perf_counter() - t0, world)
    # two steps in flight on two sets of device buffers and of pinned result buffers
    outs = [(Rh, Oh), (torch.empty_like(Rh).pin_memory(), torch.empty_like(Oh).pin_memory())]
    for i in range(6):
        arena.pipelined_wait(i & 1)
        arena.linalg_pipelined(kind, vh, uh, outs[i & 1][0], outs[i & 1][1], chunks=4, slot=i & 1, wait=False)
    arena.pipelined_wait(0)
    arena.pipelined_wait(1)
    t0 = _wall_start(torch, world)
    for i in range(steps):
        arena.pipelined_wait(i & 1)
        arena.linalg_pipelined(kind, vh, uh, outs[i & 1][0], outs[i & 1][1], chunks=4, slot=i & 1, wait=False)
    arena.pipelined_wait(0)
    arena.pipelined_wait(1)
    dt = _wall_max(torch, time.perf_counter() - t0, world)
    same = bool(torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]))
    return {"value": world * arena.n_rows_total * steps / dt, "unit": "rows/s",
            "serial_value": world * arena.n_rows_total * steps / dt_serial,
            "h2d_bytes_per_step": 8 * (vh.numel() + uh.numel()), "d2h_bytes_per_step": 8 * (Rh.numel() + Oh.numel()),
            "api": "paper_1702_06943_b200.arena.BlockArena.linalg_pipelined (arena and slot cache resident, built once; "
                   "4 slices: u upload, fused launch and R/O read-back overlap on three streams, the step replayed "
                   "as one CUDA graph; value: two steps in flight on two buffer sets, serial_value: one at a time)",
            "both_slots_bit_identical": same,
            "note": "operands in, results out per step; the headline e2e above streams the TOC1 blocks too"}


def run_reference(args, rank, world):
    """The reference arm: the CPU oracle port on this host's cores (rank 0 only)."""
    if rank != 0:
        return
    from oracle import oracle as O

    O.build()
    nb = args.batches_per_gpu
    rp, c, vals, batch_row = make_shard(0, nb)
    trees = []
    for b in range(nb):
        lo, hi = rp[batch_row[b]], rp[batch_row[b + 1]]
        enc = O.encode_csr(COLS, rp[batch_row[b] : batch_row[b + 1] + 1] - lo, c[lo:hi], vals[lo:hi])
        trees.append(O.Tree.from_encoding(enc))
    rng = np.random.default_rng(np.random.SeedSequence([SEED, 7, 0]))
    v = rng.standard_normal(COLS)
    u = rng.standard_normal(nb * ROWS)
    row_base = np.arange(nb, dtype=np.int64) * ROWS
    threads = O.max_threads()
    k = min(32, nb)
    t0 = time.perf_counter()
    O.sweep(trees[:k], row_base[:k], v, u, 2, threads)
    per_batch = max((time.perf_counter() - t0) / k, 1e-7)
    budget = 90.0
    sample = int(max(1, min(nb, budget / max(args.steps + args.warmup, 1) / per_batch)))
    for _ in range(args.warmup):
        O.sweep(trees[:sample], row_base[:sample], v, u, 2, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.sweep(trees[:sample], row_base[:sample], v, u, 2, threads)
    dt = time.perf_counter() - t0
    value = sample * ROWS * args.steps / dt
    desc = (f"oracle port (C restatement of reference kernels.py:115-174, OpenMP {threads} threads): A.v+v^T.A over "
            f"the first {sample} of {nb} config-2 batches per step, trees prebuilt (cli.py:316-317)")
    emit({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-2 generator, seeded)",
        "config": {"workload": f"config 2 sweep: {nb} TOC-compressed 250x784 f64 mini-batches; step = A.v and v^T.A",
                   "batches_per_gpu": nb, "rows_per_batch": ROWS, "n_cols": COLS},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


if __name__ == "__main__":
    main()
