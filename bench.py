#!/usr/bin/env python
"""Benchmark: ms per forward Zbc x + adjoint Zbc^H y on the Tucker-compressed
1 mm-class PWL coupling matrix (BASELINE.json configs[3], "c4"), on N B200s.

One step = one forward and one adjoint over the whole store, x and Phi
resident in HBM (value), and the same pair through the public API with host
buffers (e2e).  Multi-GPU: one process per GPU (torchrun), columns sharded by
cost; NCCL reduce of y, NCCL all-gather of z; time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
  python bench.py --impl reference ...     # the CPU reference (restated, oracle/)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 1234  # reference default seed (include/tuckmat/experiments.hpp:51); Phi uses SEED + 1


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-cols", type=int, default=0, help="columns in the CPU sample (0 = auto)")
    ap.add_argument("--shard", default="rows", choices=["rows", "columns"],
                    help="N > 1: row-slab pieces (SURVEY §8e, no forward reduction) or column ranges")
    return ap.parse_args()


# ------------------------------------------------------------------ utilities --
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a moment to start: wait for its first line so a
            # short timed region is still sampled, then keep only in-region lines
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.02)
            self.lines = []
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if not self.lines:  # region shorter than one period: one more sample at its end
            t0 = time.time()
            while not self.lines and time.time() - t0 < 0.5:
                time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            try:
                pw.append(float(parts[3]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def committed_traffic(cfg):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/traffic.json), when it was
    taken on this config; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    if not cfg.name.startswith(t.get("config", "") + ":"):
        return None
    v = t.get("dram_bytes_per_launch") or []
    return int(sum(v) / len(v)) if v else None


def f16_peak_tflops(torch):
    """cuBLAS fp16 GEMM 8192^3 throughput measured in this run (best of 5),
    beside MEASURED_PEAKS.json's bf16 figures (same tensor-core rate)."""
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=torch.float16)
    b = torch.randn(n, n, device="cuda", dtype=torch.float16)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    return best


def fp64_peak_tflops(torch):
    """cuBLAS DGEMM 8192^3 throughput (best of 5): the FP64 roofline
    denominator of the complex128 (CUDA-core DFMA) kernels."""
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=torch.float64)
    b = torch.randn(n, n, device="cuda", dtype=torch.float64)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    return best


def fp32_peak_tflops(torch, tf32=False):
    """cuBLAS SGEMM 8192^3 throughput (best of 5): plain FP32 (FFMA) or with
    TF32 tensor cores — the roofline denominators the driver does not measure
    (MEASURED_PEAKS.json has HBM and bf16 only)."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = tf32
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        for _ in range(2):
            a @ b
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            e1.synchronize()
            best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        del a, b
        return best
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


# ------------------------------------------------------------- CPU reference --
def ref_store(kind, cfg, ranks, payload, v=None, tmpdir=None):
    """The CPU store of the reference arm / cpu_baseline: the reference itself
    (oracle/_ref: proj/src compiled unchanged, kind "reference") when it was
    built, else the restatement (oracle/, kind "port").  ACA stores go
    through the reference's own CTA1 loader."""
    from oracle import oracle as O
    nc = np.asarray(ranks).shape[0]
    if kind == "reference":
        from oracle import ref as R
        if v is None:
            return R.RefCC.from_compressed(O.Compressed(cfg.grid, cfg.q, nc, ranks, payload))
        path = os.path.join(tmpdir, "store.cta1")
        O.save_cta1(path, O.Aca(cfg.grid, cfg.q, ranks, payload, v), 1.0, 0)
        return R.RefAca.load_cta1(path)
    if v is None:
        return O.OracleStore(O.Compressed(cfg.grid, cfg.q, nc, ranks, payload))

    class _PortAca:  # aca_forward / aca_adjoint of the restatement (oracle.py)
        def __init__(self):
            self.fac = O.Aca(cfg.grid, cfg.q, ranks, payload, v)

        def aca_forward(self, x, w):
            return O.aca_forward(self.fac, x, w)

        def aca_adjoint(self, phi, w):
            return O.aca_adjoint(self.fac, phi, w)
    return _PortAca()


def ref_kind():
    try:
        from oracle import ref as R
        return "reference" if R.available() else "port"
    except Exception:
        return "port"


def full_cpu_pair(cfg):
    """Configs whose whole reference product pair takes seconds on the host
    are timed in full; the large ones (c4, c5) through the bounded sample."""
    from paper_2103_06393_b200.sharded import column_costs
    from paper_2103_06393_b200.workloads import rank_table
    return float(column_costs(cfg.grid, rank_table(cfg, SEED), cfg.p).sum()) < 2e11


def sample_columns(cfg, ranks, n):
    """The CPU legs' column sample: the n columns whose per-column madd count is
    closest to the median, in column order.  A sample of near-equal columns
    keeps the W workers of the timed rounds equally busy, as the whole store's
    thousands of columns do under the reference's dynamic column queue
    (src/matvec.cpp:34,40-42); the first n columns (ranks varying 9-12 at
    config 4) left workers idle at the end of every round and overestimated
    the adjoint by ~25 %."""
    from paper_2103_06393_b200.sharded import column_costs
    costs = column_costs(cfg.grid, ranks, cfg.p)
    n = min(int(n), len(costs))
    return np.sort(np.argsort(np.abs(costs - np.median(costs)), kind="stable")[:n])


def column_payload(cfg, ranks, payload, cols):
    """The payload slices of columns `cols` (all q components each), concatenated
    (numpy or torch payload of the whole store, [col][comp] tensor order)."""
    from paper_2103_06393_b200.workloads import tensor_offsets
    off = tensor_offsets(cfg.grid, ranks)
    q = cfg.q
    parts = [payload[int(off[j * q]):int(off[(j + 1) * q])] for j in cols]
    if isinstance(payload, np.ndarray):
        return np.concatenate(parts)
    import torch
    return torch.cat(parts)


def cpu_sample(cfg, ranks, host_payload_fn, x_full, phi_full, ncols_sample, workers, kind="port", fixed=None):
    """Time the reference's forward + adjoint (src/matvec.cpp:17-102) on a
    balanced sample of `ncols_sample` columns (sample_columns) with `workers`
    host threads, and scale to the whole store by the algorithmic madd count.
    host_payload_fn(sel) returns the payload of columns `sel`.  Both products
    are modelled as a fixed per-call cost + rounds of W columns at a constant
    rate, fitted on W and 2W columns; with `fixed` ({"fwd": s, "adj": s} from
    earlier calls) only the 2W-column store is timed (the reference arm's
    timed steps)."""
    from paper_2103_06393_b200.sharded import column_costs

    from paper_2103_06393_b200.workloads import tensor_offsets

    sel = sample_columns(cfg, ranks, ncols_sample)
    pay = host_payload_fn(sel)  # complex128 (already c64-rounded values)
    costs_all = column_costs(cfg.grid, ranks, cfg.p)
    rs, costs, xs = ranks[sel], costs_all[sel], x_full[sel]

    def timed_forward(nc):
        off = tensor_offsets(cfg.grid, rs[:nc])
        st = ref_store(kind, cfg, rs[:nc], pay[: int(off[-1])])
        t0 = time.perf_counter()
        st.forward(np.asfortranarray(xs[:nc]), workers)
        return time.perf_counter() - t0, st

    def timed_adjoint(st):
        t0 = time.perf_counter()
        st.adjoint(phi_full, workers)
        return time.perf_counter() - t0

    # stacked_forward with W workers = a fixed cost (zeroing and serially
    # summing the W rows x p partials, src/matvec.cpp:30-38,58-59) + rounds of
    # W columns in parallel; stacked_adjoint = a fixed per-call cost (the
    # q n_v x p Phi block handed over, the output) + rounds of W columns.  Time
    # W and 2W columns with the same W workers: the difference is one round of
    # column work at full thread occupancy.
    def fit(ta, tb, ca, cb, fx):
        if fx is not None:  # two rounds of W columns against the calibrated fixed cost
            rate = cb / max(tb - fx, 1e-9)
            return rate, fx
        rate = (cb - ca) / max(tb - ta, 1e-9) if cb > ca else cb / tb  # madds per second, all workers
        return rate, max(ta - ca / rate, 0.0)

    W = workers
    n1, n2 = min(W, ncols_sample), min(2 * W, ncols_sample)
    ca, cb = costs[:n1].sum(), costs[:n2].sum()
    if fixed is None:
        ta, st_a = timed_forward(n1)
        tb, st = timed_forward(n2)
        aa, ab = timed_adjoint(st_a), timed_adjoint(st)
        del st_a
        rf, ff = fit(ta, tb, ca, cb, None)
        ra, fa = fit(aa, ab, ca, cb, None)
    else:
        tb, st = timed_forward(n2)
        ab = timed_adjoint(st)
        rf, ff = fit(None, tb, ca, cb, fixed["fwd"])
        ra, fa = fit(None, ab, ca, cb, fixed["adj"])
    total = costs_all.sum()
    return {"fwd_s": ff + total / rf, "adj_s": fa + total / ra, "scale": float(total / cb), "fwd_fixed_s": ff,
            "adj_fixed_s": fa}


def cpu_full(cfg, ranks, payload, v, x, phi, workers, kind, repeats=1):
    """The whole reference product pair (forward + adjoint, or the ACA pair)
    timed with wall clock as run_matvec_bench does (src/experiments.cpp:530-535)."""
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        st = ref_store(kind, cfg, ranks, payload, v, td)
        tf, ta = [], []
        for _ in range(repeats):
            t0 = time.perf_counter()
            st.aca_forward(x, workers) if v is not None else st.forward(x, workers)
            t1 = time.perf_counter()
            st.aca_adjoint(phi, workers) if v is not None else st.adjoint(phi, workers)
            t2 = time.perf_counter()
            tf.append(t1 - t0)
            ta.append(t2 - t1)
    return {"fwd_s": statistics.median(tf), "adj_s": statistics.median(ta)}


def cpu_workers(cfg, ncols_cap):
    nproc = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    rows = cfg.q * int(np.prod(cfg.grid))
    # stacked_forward holds one rows x p complex128 partial + one decompressed tensor per worker
    per_worker = 16 * rows * cfg.p + 3 * 16 * int(np.prod(cfg.grid)) + (64 << 20)
    budget = max(1, int((avail - 8 * 16 * rows) // per_worker))
    return max(1, min(nproc, budget, ncols_cap))


FULL_CPU_FILES = ("r02_cpu_full.jsonl", "r02t_cpu_full.jsonl")


def full_measurement(cfg):
    """The committed full-size measurements of the reference on GPU-box hosts
    (tools/cpu_reference.py -> profiles/r02*_cpu_full.jsonl): the latest full
    run of this config, with every full run's pair time in "all_pair_s" and
    the sample model of the latest line that has one."""
    runs, model = [], None
    for fn in FULL_CPU_FILES:
        try:
            with open(os.path.join(ROOT, "profiles", fn)) as f:
                for ln in f:
                    d = json.loads(ln)
                    if d.get("config") != cfg.name:
                        continue
                    if d.get("repeats", 1) > 0:
                        runs.append(d)
                    if d.get("sample_model"):
                        model = d["sample_model"]
        except (OSError, ValueError):
            continue
    if not runs:
        return None
    out = dict(runs[-1])
    out["all_pair_s"] = [r["pair_s"] for r in runs]
    if model is not None:
        out["sample_model"] = model
    return out


def config_dict(cfg, world, shard="rows"):
    """The workload description both arms print (same dict: same_config)."""
    from paper_2103_06393_b200.workloads import rank_table
    gb = compressed_bytes(cfg, rank_table(cfg, SEED)) / 1e9
    return {"workload": cfg.name, "grid": list(cfg.grid), "q": cfg.q, "m": cfg.m, "p": cfg.p,
            "aca_m2": cfg.aca_m2 or None,
            "parallelism": f"row-slab-shard x{world}" if world > 1 and shard == "rows" else f"column-shard x{world}",
            "l2": "inputs larger than L2 (compressed store %.2f GB c64 + derived tensor-core operands)" % gb
            if gb >= 0.2 else "L2 flushed between timed steps (512 MB write outside the step events; store %.3f GB)"
            % gb}


# --------------------------------------------------------------------- main --
def run_reference(args):
    """--impl reference: the reference's own CPU matvec path on the host cores
    (oracle/_ref, proj/src compiled unchanged; the restatement oracle/ only if
    that was not built), same config / metric as the GPU arm.  Small configs
    run whole; config 4 / 5 run the bounded sample and extrapolate, with the
    model's error against a committed full-size run reported beside it."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2103_06393_b200.workloads import CONFIGS, rank_table, synthetic_v, tensor_scales

    cfg = CONFIGS[args.config]
    kind = ref_kind()
    ranks = rank_table(cfg, SEED)
    scales = tensor_scales(cfg, SEED)
    nrows = cfg.q * int(np.prod(cfg.grid))
    full = full_cpu_pair(cfg)
    W = cpu_workers(cfg, 64 if full else 32)
    ncs = args.cpu_cols or 2 * W
    rnd = (lambda a: a.astype(np.complex64).astype(np.complex128)) if cfg.dtype == "c64" else (lambda a: a)
    x = rnd(cn01(cfg.aca_m2 or cfg.m, cfg.p, SEED))
    phi = np.asfortranarray(rnd(cn01(nrows, cfg.p, SEED + 1)))
    times = []
    if full:
        pay = _numpy_synthetic(cfg, ranks, scales, SEED)
        v = rnd(synthetic_v(cfg, SEED)) if cfg.aca_m2 else None
        for s in range(args.warmup + args.steps):
            r = cpu_full(cfg, ranks, pay, v, x, phi, W, kind)
            if s >= args.warmup:
                times.append((r["fwd_s"] + r["adj_s"]) * 1e3)
        sample = f"the whole product pair ({cfg.m} columns x {cfg.q} components, p = {cfg.p}) with {W} worker threads"
    else:
        sel = sample_columns(cfg, ranks, ncs)
        pay = _numpy_synthetic(cfg, ranks[sel], scales[sel], SEED)
        fixed, fixes, afixes = None, [], []
        for s in range(args.warmup + args.steps):
            # warm-up steps calibrate the forward's fixed partial-sum cost (W and 2W
            # columns); each timed step then runs one round of W columns
            r = cpu_sample(cfg, ranks, lambda sel_: pay, x, phi, ncs, W, kind, None if s < args.warmup else fixed)
            if s < args.warmup:
                fixes.append(r["fwd_fixed_s"])
                afixes.append(r["adj_fixed_s"])
                fixed = {"fwd": statistics.median(fixes), "adj": statistics.median(afixes)}
            else:
                times.append((r["fwd_s"] + r["adj_s"]) * 1e3)
        sample = (f"per step the forward on {ncs} of {cfg.m} columns (the median-cost ones, all q={cfg.q} components, two rounds of {W} "
                  f"worker threads) and the adjoint on the same {ncs} columns, each extrapolated as its fixed "
                  f"per-call cost (median of the warm-up steps' two-point fits on {W} and {ncs} columns) + the "
                  f"per-round rate x the store's madd count")
    ms = statistics.median(times)
    line = {
        "impl": "reference", "metric": metric_name(cfg), "value": round(ms, 1), "unit": "ms", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 1), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "c128 (the reference's arithmetic; c64-rounded factors)", "data": "synthetic",
        "config": config_dict(cfg, world, args.shard),
        "cpu_baseline": {"value": round(ms, 1), "unit": "ms", "cores": W, "kind": kind, "sample": sample},
        "e2e": {"value": round(ms, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated": not full,
    }
    fm = full_measurement(cfg)
    if fm:
        line["full_size_measurement"] = {"pair_ms": round(fm["pair_s"] * 1e3, 1), "workers": fm["workers"],
                                         "all_pair_ms": [round(v * 1e3, 1) for v in fm["all_pair_s"]],
                                         "cpu": fm.get("cpu"), "source": "profiles/r02*_cpu_full.jsonl"}
        if not full:
            line["full_size_measurement"]["sample_model_rel_error"] = (fm.get("sample_model") or {}).get(
                "rel_error_vs_full")
            line["full_size_measurement"]["note"] = (
                "full-size runs of the same store on GPU-box hosts; the sample model's error against the same "
                "host's full run is sample_model_rel_error (single samples scatter by about 15 %, DESIGN.md §7)")
    print(json.dumps(line), flush=True)


def _numpy_synthetic(cfg, ranks, scales, seed):
    """Host copy of the synthetic store's first columns, c64-rounded (for the
    CPU legs without a GPU-generated payload)."""
    import torch
    from paper_2103_06393_b200.workloads import synthetic_payload
    pay, _ = synthetic_payload(cfg.grid, ranks, scales, seed + 1000, device="cpu")
    if cfg.dtype == "c64":
        pay = pay.to(torch.complex64).to(torch.complex128)
    return pay.cpu().numpy()


def cn01(rows, cols, seed):
    """Seeded CN(0,1) block, column-major."""
    rng = np.random.default_rng(seed)
    a = (rng.standard_normal((rows, cols)) + 1j * rng.standard_normal((rows, cols))) / math.sqrt(2)
    return np.asfortranarray(a)


def compressed_bytes(cfg, ranks, n1=None):
    """Bytes of the compressed store proper (cores + factors, c64): the
    roofline's B_alg term, without the derived tensor-core
    operand copies.  n1: the grid height of a row-slab piece."""
    r = np.asarray(ranks, np.int64).reshape(-1, 3)
    n1, n2, n3 = (cfg.grid[0] if n1 is None else n1), cfg.grid[1], cfg.grid[2]
    scalars = (r[:, 0] * r[:, 1] * r[:, 2] + n1 * r[:, 0] + n2 * r[:, 1] + n3 * r[:, 2]).sum()
    return int(scalars) * (8 if cfg.dtype == "c64" else 16)


def metric_name(cfg):
    return f"ms per Zbc*x + Zbc^H*y matvec pair ({cfg.name})"


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # TMB_BENCH_SMOKE_1GPU=1: a functional check of the N > 1 code path on a
    # one-GPU box (every rank on cuda:0, gloo collectives); never a measurement.
    smoke1 = os.environ.get("TMB_BENCH_SMOKE_1GPU", "0") == "1"
    if smoke1:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if smoke1:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2103_06393_b200 import DeviceStore, launch_count
    from paper_2103_06393_b200.sharded import (RowShardedStore, ShardedStore, balanced_shards, column_costs,
                                               component_costs, row_pieces, slice_payload_rows)
    from paper_2103_06393_b200.workloads import CONFIGS, rank_table, synthetic_payload, synthetic_v, tensor_scales

    cfg = CONFIGS[args.config]
    ranks = rank_table(cfg, SEED)
    scales = tensor_scales(cfg, SEED)
    costs = column_costs(cfg.grid, ranks, cfg.p)
    aca = bool(cfg.aca_m2)  # ACA configs: aca_forward / aca_adjoint (src/matvec.cpp:150-175), V included
    v_all = synthetic_v(cfg, SEED) if aca else None
    rows_mode = world > 1 and args.shard == "rows"
    shards = balanced_shards(costs, world)
    c0, c1 = (0, cfg.m) if rows_mode else shards[rank]  # rows mode: every rank holds all columns of its pieces
    nrows = cfg.q * int(np.prod(cfg.grid))
    cdt = torch.complex64 if cfg.dtype == "c64" else torch.complex128

    # --- store: seeded synthetic payload generated on the device, packed once --
    t_build = time.perf_counter()
    if rows_mode:
        # this rank's (component, i1-slab) pieces, each a one-component store on
        # its sub-grid with every column (sharded.row_pieces / slice_payload_rows)
        r1max = int(ranks[..., 0].max())
        layout = row_pieces(component_costs(cfg.grid, ranks, cfg.p), cfg.grid[0], world, align=8,
                            min_rows=8 * ((r1max + 7) // 8))
        pieces = []
        for k, a, b in layout[rank]:
            rk = np.ascontiguousarray(ranks[:, k:k + 1, :])
            payk, _ = synthetic_payload(cfg.grid, rk, scales[:, k:k + 1], SEED + 1000 + 7 * k, device=dev)
            payp = slice_payload_rows(cfg.grid, rk, payk, a, b)
            del payk
            pieces.append((k, a, b, DeviceStore.from_arrays((b - a, cfg.grid[1], cfg.grid[2]), 1, rk, payp, cfg.dtype,
                                                            local, v=v_all if aca else None)))
            del payp
        part_stores = [st for *_, st in pieces]
        store = part_stores[0] if part_stores else None
    else:
        pay, _ = synthetic_payload(cfg.grid, ranks[c0:c1], scales[c0:c1], SEED + 1000 + c0, device=dev)
        store = DeviceStore.from_arrays(cfg.grid, cfg.q, ranks[c0:c1], pay, cfg.dtype, local,
                                        v=v_all[:, c0:c1] if aca else None)
        part_stores = [store]
    cpu_pay = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if full_cpu_pair(cfg):
            cpu_pay = pay.to(cdt).to(torch.complex128).cpu().numpy()
        else:
            W = cpu_workers(cfg, 32)
            ncs = min(args.cpu_cols or 2 * W, c1 - c0)
            sel = sample_columns(cfg, ranks, ncs)
            cpu_pay = column_payload(cfg, ranks, pay, sel).to(cdt).to(torch.complex128).cpu().numpy()
    if not rows_mode:
        del pay
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build
    if rows_mode:
        sh = RowShardedStore(pieces, cfg.grid, cfg.q, cfg.m, layout, m2=cfg.aca_m2 or 0)
    else:
        sh = ShardedStore(store, c0, c1, cfg.m, shards=shards)

    # --- inputs: CN(0,1), seeded (x: numpy, Phi: device RNG) ---------------------
    x_host = cn01(cfg.aca_m2 or cfg.m, cfg.p, SEED).astype(np.complex64 if cfg.dtype == "c64" else np.complex128)
    x = torch.from_numpy(np.ascontiguousarray(x_host.T)).to(dev).t()
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + 1)
    phi = (torch.randn((cfg.p, nrows), dtype=cdt, device=dev, generator=g)).t()
    xs = x if aca else x[c0:c1]

    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        y = sh.aca_forward(xs) if aca else sh.forward(xs)
        if ev:
            ev[1].record(stream)
        z = sh.aca_adjoint(phi) if aca else sh.adjoint(phi)
        if ev:
            ev[2].record(stream)
        return y, z

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    peaks = measured_peaks()
    fp32_peak = fp32_peak_tflops(torch) if rank == 0 else None
    f16_peak = f16_peak_tflops(torch) if rank == 0 else None
    fp64_peak = fp64_peak_tflops(torch) if rank == 0 else None
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    if rank == 0:
        clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    torch.cuda.profiler.start()  # ncu --profile-from-start off captures exactly the timed region
    l0 = launch_count()
    t_all0 = torch.cuda.Event(enable_timing=True)
    t_all1 = torch.cuda.Event(enable_timing=True)
    # stores smaller than L2 (126 MB): flush L2 between timed steps (a 512 MB
    # write, outside the per-step events) so each step re-reads its operands
    flush = compressed_bytes(cfg, ranks) < (200 << 20)
    fbuf = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    t_all0.record(stream)
    for s in range(args.steps):
        if flush:
            fbuf.fill_(s & 0xFF)
        step(evs[s])
    t_all1.record(stream)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    if world > 1:
        dist.barrier()
    launches = launch_count() - l0
    clk = clocks.stop() if rank == 0 else None
    total_ms = t_all0.elapsed_time(t_all1)
    fwd_ms = [e[0].elapsed_time(e[1]) for e in evs]
    adj_ms = [e[1].elapsed_time(e[2]) for e in evs]
    t = torch.tensor([total_ms, statistics.median(fwd_ms), statistics.median(adj_ms)], device=dev,
                     dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, fwd_med, adj_med = t.tolist()
    if flush:  # the per-step events exclude the L2 flushes
        tt = torch.tensor([sum(f + a for f, a in zip(fwd_ms, adj_ms))], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = tt.item()
    ms_per_step = total_ms / args.steps

    # --- e2e through the public API with host buffers ---------------------------
    e2e = None
    if not args.no_e2e:
        import ctypes
        from paper_2103_06393_b200._lib import TM_HOST, lib
        from paper_2103_06393_b200.matvec import _check
        npdt = np.complex64 if cfg.dtype == "c64" else np.complex128
        xin = x_host if aca else x_host[c0:c1]
        xh = torch.from_numpy(np.asfortranarray(xin).ravel(order="F")).pin_memory()
        yh = torch.empty(nrows * cfg.p, dtype=cdt).pin_memory()
        ph = phi.t().contiguous().cpu().pin_memory()  # every rank reads the whole Phi
        zrows = cfg.aca_m2 if aca else c1 - c0
        zh = torch.empty(zrows * cfg.p, dtype=cdt).pin_memory()
        e2e_times = []
        h2d = d2h = 0
        for s in range(1 + args.e2e_steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if world == 1 and aca:
                _check(lib().tm_aca_forward(store.handle, xh.data_ptr(), cfg.aca_m2, cfg.aca_m2, cfg.p, yh.data_ptr(),
                                            nrows, TM_HOST, None))
                _check(lib().tm_aca_adjoint(store.handle, ph.data_ptr(), nrows, nrows, cfg.p, zh.data_ptr(),
                                            cfg.aca_m2, TM_HOST, None))
                h2d = xh.numel() * xh.element_size() + ph.numel() * ph.element_size()
                d2h = yh.numel() * yh.element_size() + zh.numel() * zh.element_size()
            elif world == 1:
                _check(lib().tm_forward(store.handle, xh.data_ptr(), c1 - c0, c1 - c0, cfg.p, yh.data_ptr(), nrows,
                                        TM_HOST, None, None))
                _check(lib().tm_adjoint(store.handle, ph.data_ptr(), nrows, nrows, cfg.p, zh.data_ptr(), c1 - c0,
                                        TM_HOST, None, None))
                h2d = xh.numel() * xh.element_size() + ph.numel() * ph.element_size()
                d2h = yh.numel() * yh.element_size() + zh.numel() * zh.element_size()
            else:
                # sharded public API: host x -> device, forward + NCCL reduce,
                # y -> host on rank 0; host phi -> device on every rank (each
                # over its own PCIe link), adjoint + all-gather, z -> host
                xd = xh.to(dev, non_blocking=True).reshape(cfg.p, -1).t()
                y = sh.aca_forward(xd) if aca else sh.forward(xd)
                if rank == 0:
                    yh.copy_(y.t().reshape(-1) if y.dim() == 2 else y, non_blocking=True)
                pd = ph.to(dev, non_blocking=True).t()
                z = sh.aca_adjoint(pd) if aca else sh.adjoint(pd)
                zf = torch.empty(z.numel(), dtype=cdt).pin_memory()
                zf.copy_(z.t().reshape(-1) if z.dim() == 2 else z, non_blocking=True)
                torch.cuda.synchronize()
                h2d = xh.numel() * xh.element_size() + ph.numel() * ph.element_size()
                d2h = (yh.numel() * yh.element_size() if rank == 0 else 0) + zf.numel() * zf.element_size()
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            if s > 0:
                e2e_times.append(dt)
        tt = torch.tensor([statistics.median(e2e_times)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": tt.item(), "unit": "ms", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
        if world > 1:
            e2e["note"] = "multi-GPU e2e uses the sharded Python API; byte counts are rank 0's"

    sb = torch.tensor([float(sum(st.device_bytes for st in part_stores))], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(sb, op=dist.ReduceOp.SUM)
    store_bytes_all = sb.item()

    # --- roofline of the dominant kernels (one tensor-core launch per forward;
    # the adjoint is Phi split + tensor-core kernel + partial reduction) ------
    dec = acc = 0
    for st in part_stores:
        d_, a_ = st.opcounts(cfg.p)
        dec, acc = dec + d_, acc + a_
    flops = 8.0 * (dec + acc)  # OpCounts x 8 real flops per complex madd (this rank's shard)
    if aca:  # + the V side of one ACA product (V^H x or V t): m2 r_c p madds
        flops += 8.0 * cfg.aca_m2 * (c1 - c0) * cfg.p
    tc = cfg.dtype == "c64" and os.environ.get("TMB_DISABLE_TC", "0") != "1"
    roof = None
    if rank == 0:
        if tc:
            # complex64 on the tensor cores as scaled 2-term fp16 splits: every
            # fp32-equivalent real multiply-add costs three fp16 tensor-core
            # multiply-adds (hi.hi + hi.lo + lo.hi), so the compute roofline of
            # the algorithmic flops is the dense fp16/bf16 peak / 3.  The step
            # is long (hundreds of ms), so the sustained (power-capped) figure
            # of MEASURED_PEAKS.json applies.
            bf16 = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops") or 1400.0
            peak = bf16 / 3.0
            bound, unit_src = "tensor", ("measured (MEASURED_PEAKS.json bf16_tflops_sustained = %s TFLOP/s dense) / 3 "
                                         "for the 3-product fp16 split; cuBLAS fp16 GEMM in this run: %.1f TFLOP/s"
                                         % (bf16, f16_peak))
            kernels = ("fwd_tc_kernel", "adj_tc_kernel (+ absmax, adj_split_phi_kernel, adj_reduce_kernel)")
            paths = part_stores[0].kernel_paths() if part_stores else {}
            if paths.get("forward") == "tcgen05+warena":  # the W arena (DESIGN §3 / §4)
                k3w = cfg.p >= int(os.environ.get("TMB_K3_PMIN", "16")) and os.environ.get("TMB_K3", "1") != "0"
                kernels = ("fwd_k3w_kernel (K3W: GEMM1 T = W U3^T + GEMM2 Y += T X)" if k3w
                           else "fwd_tc_kernel (A operand from the W arena)", kernels[1])
            if paths.get("adjoint") == "tcgen05+gemm":
                kernels = (kernels[0], "fwd_tc_kernel<ADJ> (G = conj(W)^T Phi on the transposed W arena; "
                                       "+ adjg_split_phi_kernel, adjg_contract_kernel)")
        elif cfg.dtype == "c128":
            peak = fp64_peak
            bound, unit_src = "fp64", "measured here: cuBLAS DGEMM 8192^3 (the c128 kernels run DFMA)"
            kernels = ("fwd_cc_kernel", "adj_cc_kernel (+ adj_reduce_kernel)")
        else:
            peak = fp32_peak
            bound, unit_src = "fp32-ffma", "measured here: cuBLAS SGEMM 8192^3 without TF32"
            kernels = ("fwd_cc_kernel", "adj_cc_kernel (+ adj_reduce_kernel)")
        fa, aa = flops / (fwd_med * 1e-3) / 1e12, flops / (adj_med * 1e-3) / 1e12
        roof = {"bound": bound, "kernel": kernels[0], "achieved": round(fa, 2), "peak": round(peak, 2),
                "unit": "TFLOP/s", "frac": round(fa / peak, 4), "peak_source": unit_src, "traffic": committed_traffic(cfg),
                "traffic_unit": "bytes per launch (DRAM read + write; profiles/traffic.json)",
                "algorithmic_flops_per_launch": flops,
                "adjoint": {"kernel": kernels[1], "achieved": round(aa, 2), "frac": round(aa / peak, 4)},
                "hbm_bytes_algorithmic": int(compressed_bytes(cfg, ranks[c0:c1]) + (c1 - c0) * cfg.p * 8
                                             + nrows * cfg.p * 8) if not rows_mode else
                int(sum(compressed_bytes(cfg, ranks[:, k], n1=b - a) for k, a, b in layout[rank])
                    + cfg.m * cfg.p * 8 + sum(st.rows for st in part_stores) * cfg.p * 8),
                "hbm_peak_gbs": peaks.get("hbm_gbs"), "fp32_ffma_peak_tflops": round(fp32_peak, 2),
                "fp64_dgemm_tflops_this_run": round(fp64_peak, 2),
                "f16_gemm_tflops_this_run": round(f16_peak, 2), "bf16_peak_tflops_measured": peaks.get("bf16_tflops")}
        if world > 1:
            # SURVEY §8d multi-GPU term C_coll / BW_NVLink: the forward's reduce of the
            # q n_v x p partial y and the adjoint's all-gather of the padded z shards,
            # against the NVLink 5 per-direction figure (spec, not measured here)
            if rows_mode:  # pieces' rows of y to rank 0 + all-reduce of the m x p partial z
                cbytes = nrows * cfg.p * 8 * (world - 1) // world + 2 * (cfg.aca_m2 or cfg.m) * cfg.p * 8
            else:
                cbytes = nrows * cfg.p * 8 + world * max(b - a for a, b in shards) * cfg.p * 8
            roof["collective"] = {"bytes_per_step": int(cbytes), "nvlink_gbs_spec": 900.0,
                                  "t_roof_ms": round(cbytes / 900e9 * 1e3, 3),
                                  "note": "one GPU's compute roofline above is its shard's"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and cpu_pay is not None:
        kind = ref_kind()
        phi_h = np.asfortranarray(phi.cpu().numpy().astype(np.complex128))
        if full_cpu_pair(cfg):
            W = cpu_workers(cfg, 64)
            v64 = v_all.astype(np.complex64).astype(np.complex128) if aca and cfg.dtype == "c64" else v_all
            r = cpu_full(cfg, ranks, cpu_pay, v64, x_host.astype(np.complex128), phi_h, W, kind)
            sample = (f"the whole product pair ({cfg.m} columns x {cfg.q} components, p = {cfg.p}"
                      + (", through aca_forward / aca_adjoint" if aca else "") + f") with {W} worker threads")
            extra = {}
        else:
            W = cpu_workers(cfg, 32)
            ncs = min(args.cpu_cols or 2 * W, c1 - c0)
            r = cpu_sample(cfg, ranks, lambda sel_: cpu_pay, x_host.astype(np.complex128), phi_h, ncs, W, kind)
            sample = (f"forward timed on {W} and {ncs} of {cfg.m} columns (the median-cost ones, all {cfg.q} components) with {W} worker "
                      f"threads, and the adjoint likewise, each extrapolated as a fixed per-call cost + the per-round rate "
                      f"(two-point fit on {W} and {ncs} columns) x the store's madd count")
            extra = {"extrapolated": True, "fwd_fixed_ms": round(r["fwd_fixed_s"] * 1e3, 1),
                     "adj_fixed_ms": round(r["adj_fixed_s"] * 1e3, 1)}
            fm = full_measurement(cfg)
            if fm:
                extra["full_size_measurement"] = {"pair_ms": round(fm["pair_s"] * 1e3, 1), "workers": fm["workers"],
                                                  "all_pair_ms": [round(v * 1e3, 1) for v in fm["all_pair_s"]],
                                                  "source": "profiles/r02*_cpu_full.jsonl",
                                                  "sample_model_rel_error": (fm.get("sample_model") or {}).get(
                                                      "rel_error_vs_full")}
        cpu = {"value": round((r["fwd_s"] + r["adj_s"]) * 1e3, 1), "unit": "ms", "cores": W, "kind": kind,
               "sample": sample, "forward_ms": round(r["fwd_s"] * 1e3, 1), "adjoint_ms": round(r["adj_s"] * 1e3, 1),
               **extra}

    if rank == 0:
        line = {
            "metric": metric_name(cfg), "value": round(ms_per_step, 3), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (seeded Tucker store with the config's shape and rank distribution)",
            "config": config_dict(cfg, world, args.shard),
            "device_store_gb": round(store_bytes_all / 1e9, 2),
            "forward_ms": round(fwd_med, 3), "adjoint_ms": round(adj_med, 3),
            "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "store_build_s": round(t_build, 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
