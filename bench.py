#!/usr/bin/env python
"""bench.py -- Batch-BFS + BCTS on B200: tree nodes (expanded + evaluated)/s and root decisions/s.

Default workload = BASELINE.json's metric configuration C5: depth 4, A = 18,
one Atari-shaped root (4x84x84 uint8 frame stack), Rainbow-shaped bf16 Q-net,
BCTS correction on. One step = one full search (every SURVEY §8a row: root
row, level expansions, leaf net, backup, correction). N > 1 (torchrun): the
same single-root search split into contiguous leaf ranges, one max
all-reduce of the packed root keys (strong scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tree nodes expanded+evaluated/sec and root decisions/sec at depth 4, A=18"


def nodes_per_root(A, d, corr):
    """Algorithmic per-root counts: expanded = sum_{k=1..d} A^k,
    evaluated = A^d + [corr]*(1 + [d>=2]*A) (+1 at d=0): the BCTS terms (Eq. 5 or Lemma 2's exact
    biases alike) need the root row and, at d >= 2, the level-1 rows."""
    expanded = sum(A ** k for k in range(1, d + 1))
    evaluated = (A ** d + ((1 if corr else 0) * (1 + (A if d >= 2 else 0))) if d >= 1 else 1)
    return expanded, evaluated


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        out = {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
               "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured",
               "sm_max_mhz": d.get("sm_max_mhz", 1965.0)}
    else:
        out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback",
               "sm_max_mhz": 1965.0}
    # fp32 FMA (ALU) peak, derived: 148 SMs x 4 SMSPs x 32 FFMA lanes x 2 FLOP x max SM clock
    out["fp32_tflops"] = 148 * 128 * 2 * out["sm_max_mhz"] * 1e6 / 1e12
    return out


FP32_CLASSES = {"mlp", "expand_dnn"}      # fixed-order fmaf kernels: ALU-bound, fp32 peak


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region.

    nvidia-smi needs ~0.1-0.3 s before its first sample, longer than a default timed region, so the
    sampler is started (and its first line awaited) before the warm-up; a reader thread timestamps
    every line and mark()/unmark() bracket the timed region. The summary uses the samples taken
    inside it (plus the one just before, so a short region still has one)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.stamped, self.t0, self.t1 = device, None, [], None, None

    def _read(self):
        for line in self.proc.stdout:
            if line.strip():
                self.stamped.append((time.monotonic(), line))

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            deadline = time.monotonic() + 3.0
            while not self.stamped and time.monotonic() < deadline:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def mark(self):
        self.t0 = time.monotonic()

    def unmark(self):
        self.t1 = time.monotonic() + 0.03   # one more sampling period

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        t0 = self.t0 if self.t0 is not None else float("-inf")
        t1 = self.t1 if self.t1 is not None else float("inf")
        before = [l for t, l in self.stamped if t < t0][-1:]
        self.lines = before + [l for t, l in self.stamped if t0 <= t <= t1]

    def summary(self):
        if not getattr(self, "lines", None):
            return None
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        load = [s for s in sm if s > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def self_launch(argv, gpus):
    """`bench.py --gpus N` outside torchrun: re-run this script as N ranks (one process per GPU)
    under torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def tab_of(cfg):
    """The C1 tabular MDP (SPEC chain-grid) for TABULAR configs, else None."""
    from synth.inputs import ENV_TABULAR, chain_c1
    return chain_c1() if cfg.env == ENV_TABULAR else None


def metric_of(cfg):
    if (cfg.A, cfg.depth) == (18, 4):
        return METRIC
    return f"tree nodes expanded+evaluated/sec and root decisions/sec at depth {cfg.depth}, A={cfg.A}"


def dtype_of(cfg):
    return "bf16" if cfg.net in (3, 4) else "f32"


CORRECTION_NAMES = {0: "correction off (vanilla TS)", 1: "correction on", 2: "correction on (Lemma 2 exact biases)"}


def workload_of(cfg, n, corr=1):
    base = f"{cfg.name}: Batch-BFS+BCTS, A={cfg.A}, depth={cfg.depth}, {n} root(s), "
    cn = CORRECTION_NAMES[corr]
    if cfg.net in (3, 4):
        return base + f"{'Rainbow' if cfg.net == 4 else 'Nature'}-shaped bf16 Q-net (random init), {cn}"
    if cfg.env == 4:
        return base + ("random-DNN forward model (3x100 hidden, P:340-341) + MLP2 100-256-A fp32 leaf net "
                       f"(random init), {cn}")
    return base + f"hash env + MLP2/table leaf values, {cn}"


# ------------------------------------------------------------------ CPU oracle leg
def oracle_sample(cfg, seconds_target=12.0, threads=None):
    """Time the oracle (as it stands) on a bounded sample of the same workload:
    whole depth-2 subtrees of the first root, run across the host cores."""
    from oracle import Oracle
    threads = threads or os.cpu_count() or 1
    o = Oracle.from_config(cfg, tab=tab_of(cfg))
    root = cfg.roots(1)
    A, d = cfg.A, cfg.depth
    exp, ev = nodes_per_root(A, d, 1)
    if d < 2 or exp + ev <= 200_000:
        # small trees: whole searches of batches of roots (one root per thread)
        roots = cfg.roots(max(threads, 1))
        done, elapsed = 0, 0.0
        while elapsed < seconds_target and done < 256 * threads:
            t = time.perf_counter()
            o.search(roots, d, cfg.gamma, cfg.beta, 1, mode=0, threads=threads)
            elapsed += time.perf_counter() - t
            done += roots.shape[0]
        nodes = (exp + ev) * done
        return {"value": nodes / elapsed, "unit": "nodes/s", "cores": threads, "kind": "oracle",
                "decisions_per_s": done / elapsed,
                "sample": f"{done} whole depth-{d} searches ({cfg.name}: A={A}), plain-C DFS, {threads} threads, "
                          f"{elapsed:.1f} s"}
    per_task_nodes = (exp + A ** d) / (A * A)      # subtree share of the tree's expansions + leaf evaluations
    done_tasks, elapsed, t0 = 0, 0.0, 0
    wave = threads
    while elapsed < seconds_target and t0 < A * A:
        n = min(wave, A * A - t0)
        t = time.perf_counter()
        o.subtrees(root, d, cfg.gamma, t0, t0 + n, threads=threads)
        elapsed += time.perf_counter() - t
        done_tasks += n
        t0 += n
    nodes = per_task_nodes * done_tasks
    return {"value": nodes / elapsed, "unit": "nodes/s", "cores": threads, "kind": "oracle",
            "decisions_per_s": nodes / elapsed / (exp + ev),
            "sample": f"{done_tasks} of the {A * A} depth-2 subtrees of root 0 ({cfg.name}: A={A}, d={d}), "
                      f"plain-C DFS, {threads} threads, {elapsed:.1f} s"}


def run_reference(args, cfg, world, rank):
    if rank != 0:
        return 0
    from oracle import Oracle
    threads = os.cpu_count() or 1
    o = Oracle.from_config(cfg, tab=tab_of(cfg))
    root = cfg.roots(1)
    A, d = cfg.A, cfg.depth
    exp, ev = nodes_per_root(A, d, args.correction)
    per_task = (exp + A ** d) / (A * A)
    ntask = min(threads, A * A)
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        o.subtrees(root, d, cfg.gamma, 0, ntask, threads=threads)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            times.append(dt)
    step = sum(times) / len(times)
    value = per_task * ntask / step
    line = {"impl": "reference", "metric": metric_of(cfg), "value": value, "unit": "nodes/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "decisions_per_s": value / (exp + ev), "metric_note": metric_of(cfg),
            "config": {"workload": workload_of(cfg, cfg.n_roots, args.correction) + f"; each step = {ntask} depth-2 subtrees "
                                   "(bounded sample)",
                       "roots": cfg.n_roots, "depth": d, "A": A},
            "cpu_baseline": {"value": value, "unit": "nodes/s", "cores": threads, "kind": "oracle",
                             "sample": f"{ntask} of {A * A} depth-2 subtrees per step, plain-C DFS (fp64, bf16-emulated net)"},
            "e2e": {"value": value, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--roots", type=int, default=0, help="override n_roots (throughput variants)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--simt", action="store_true", help="SIMT reference net (no tensor cores)")
    ap.add_argument("--tf32", action="store_true",
                    help="BCTS_F_TF32: DNN forward model / MLP2 on tcgen05 kind::tf32 (within the tf32 tolerance)")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--correction", type=int, choices=(0, 1, 2), default=1,
                    help="correction_on: 0 vanilla TS, 1 BCTS Eq. 5 (the headline), 2 Lemma 2 exact biases (NEXT-2)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(sys.argv[1:], args.gpus)

    from synth.inputs import config
    import dataclasses
    cfg = config(args.config)
    if args.roots:
        cfg = dataclasses.replace(cfg, n_roots=args.roots)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        return run_reference(args, cfg, world, rank)

    import numpy as np
    import torch
    import paper_2107_01715_b200 as P
    from paper_2107_01715_b200.parallel import world_handle
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    flags = (P.F_SIMT_NET if args.simt else 0) | (P.F_TF32 if args.tf32 else 0)
    # world > 1: every rank's handle owns an NCCL communicator (id made on rank 0, broadcast); the
    # search is then collective inside the library: each rank scores its leaf range and one
    # ncclAllReduce(MAX) of the packed root keys runs on the handle's stream
    h = world_handle(cfg, tab=tab_of(cfg), device=local, flags=flags)
    n, d, A, corr = cfg.n_roots, cfg.depth, cfg.A, args.correction
    roots_np = cfg.roots()
    roots = torch.from_numpy(roots_np.view(np.uint8).reshape(n, -1).copy()).to(dev)
    act = torch.empty(n, dtype=torch.int32, device=dev)
    q = torch.empty(n, A, dtype=torch.float32, device=dev)
    launches_per_step = [0]

    def step():
        out = h.search(roots, n, d, cfg.gamma, cfg.beta, corr, out={"actions": act, "root_q": q})
        launches_per_step[0] = out["stats"]["kernel_launches"]
        return out

    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    clk = ClockSampler(local).__enter__()   # started before the warm-up (see ClockSampler)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # ---- timed region: K steps, L2 flushed (256 MiB write, untimed) before each.
    # No per-kernel profiling inside it (event records between kernels perturb
    # the step); the per-kernel roofline comes from a profiled repeat below.
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    clk.mark()
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(i & 0xFF)
        evs[i][0].record()
        step()
        evs[i][1].record()
    torch.cuda.synchronize()
    clk.unmark()
    clk.__exit__(None, None, None)
    barrier()
    # ---- profiled repeat of the timed region: per-kernel-class CUDA events on the launching stream
    h.profile(True)
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(i & 0xFF)
        step()
    torch.cuda.synchronize()
    prof = h.profile_read()
    h.profile(False)
    step_ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([step_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = float(t.item())
    exp, ev = nodes_per_root(A, d, corr)
    total_nodes = n * (exp + ev)
    value = total_nodes / (step_ms / 1e3)

    # ---- roofline of the dominant kernel class (events on the launching stream)
    peaks = load_peaks()
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else None
    roofline = None
    kernels = {}
    step_kernel_ms = sum(v["ms"] for v in prof.values())
    for name, v in prof.items():
        per_launch_ms = v["ms"] / max(v["launches"], 1)
        ach = v["work"] / (v["ms"] / 1e3) / (1e9 if v["unit"] == "byte" else 1e12) if v["ms"] > 0 else 0.0
        kernels[name] = {"launches_per_step": v["launches"] / args.steps, "ms_per_launch": per_launch_ms,
                         "share": v["ms"] / step_kernel_ms if step_kernel_ms else 0.0,
                         "achieved": ach, "unit": "GB/s" if v["unit"] == "byte" else "TFLOP/s"}
        if v.get("big_launches") and v["big_launches"] < v["launches"] and v["big_ms"] > 0:
            # the class's largest launches alone (e.g. the deepest expanded level, the full batches)
            kernels[name]["largest"] = {
                "launches_per_step": v["big_launches"] / args.steps,
                "ms_per_launch": v["big_ms"] / v["big_launches"],
                "achieved": v["big_work"] * v["big_launches"] / (v["big_ms"] / 1e3)
                / (1e9 if v["unit"] == "byte" else 1e12)}
    if dom:
        name, v = dom
        # a kernel inside a long step (or a long timed region) runs at the power-capped sustained
        # clock: compare it with the sustained peak (MEASURED_PEAKS.json, 4 s back-to-back GEMMs)
        long_run = step_ms > 50.0 or step_ms * args.steps > 1000.0
        if v["unit"] == "byte":
            peak, unit, bound = peaks["hbm_gbs"], "GB/s", "hbm"
            psrc = peaks["source"] + " burst"
        elif args.simt or (name in FP32_CLASSES and not args.tf32):
            peak, unit, bound = peaks["fp32_tflops"], "TFLOP/s", "alu"
            psrc = f"derived: 148 SMs x 128 FP32 FMA lanes x 2 x {peaks['sm_max_mhz']:.0f} MHz"
        else:
            peak = peaks["bf16_tflops_sustained"] if long_run else peaks["bf16_tflops"]
            unit, bound = "TFLOP/s", "tensor"
            psrc = peaks["source"] + (" sustained" if long_run else " burst")
            if args.tf32 and name in FP32_CLASSES:   # kind::tf32 runs at half the bf16 rate (nominal ratio)
                peak *= 0.5
                psrc += " bf16 peak x 0.5 (tf32)"
        ach = kernels[name]["achieved"]
        # nominal denominators beside the measured ones: 2.25 PFLOP/s dense bf16,
        # 8 TB/s HBM3e; the ALU peak is already the nominal unit count x clock
        nominal = {"tensor": 1125.0 if (args.tf32 and name in FP32_CLASSES) else 2250.0, "hbm": 8000.0,
                   "alu": peaks["fp32_tflops"]}[bound]
        roofline = {"kernel": name, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                    "frac": ach / peak, "traffic": None,
                    "work_per_launch": v["work"] / max(v["launches"], 1), "peak_source": psrc,
                    "peak_nominal": nominal, "frac_nominal": ach / nominal}
        tr = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr):
            # one ncu --set full capture of this kernel (cold cache, a full launch), scaled to the
            # average timed launch by algorithmic work; unit = bytes per launch like `achieved`
            ent = json.load(open(tr)).get(cfg.name, {}).get(name)
            if ent:
                per_launch = v["work"] / max(v["launches"], 1)
                roofline["traffic"] = ent["dram_bytes_per_launch"] * per_launch / ent["work_per_launch"]
                roofline["traffic_unit"] = "bytes/launch (DRAM read+write)"
                roofline["traffic_source"] = ent["source"]

    # ---- end to end: host roots in (pinned), host outputs out, through the public API
    e2e = None
    pin_roots = torch.from_numpy(roots_np.view(np.uint8).reshape(n, -1).copy()).pin_memory()
    pin_act = torch.empty(n, dtype=torch.int32).pin_memory()
    pin_q = torch.empty(n, A, dtype=torch.float32).pin_memory()
    e2e_times = []
    for i in range(args.warmup + args.steps):
        if flush is not None:
            flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        h.search_host(pin_roots, n, d, cfg.gamma, cfg.beta, corr, pin_act, pin_q)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_times.append(dt)
    e2e_s = sum(e2e_times) / len(e2e_times)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": total_nodes / e2e_s, "unit": "nodes/s", "h2d_bytes_per_step": int(pin_roots.numel()),
           "d2h_bytes_per_step": int(pin_act.numel() * 4 + pin_q.numel() * 4), "ms_per_step": e2e_s * 1e3,
           "decisions_per_s": n / e2e_s,
           # this rank's per-call wall times (the value above is their mean, max over ranks)
           "ms_median": float(np.median(e2e_times)) * 1e3, "ms_min": min(e2e_times) * 1e3,
           "ms_max": max(e2e_times) * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(cfg)
        # the canonical CPU baseline of SURVEY §8d: the same DFS on ONE thread (smaller sample)
        one = oracle_sample(cfg, seconds_target=5.0, threads=1)
        cpu["single_thread"] = {"value": one["value"], "unit": one["unit"], "cores": 1,
                                "decisions_per_s": one["decisions_per_s"], "sample": one["sample"]}

    if rank == 0:
        line = {"metric": metric_of(cfg), "value": value, "unit": "nodes/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "tf32" if (args.tf32 and cfg.net not in (3, 4)) else dtype_of(cfg), "data": "synthetic",
                "decisions_per_s": n / (step_ms / 1e3),
                "config": {"workload": workload_of(cfg, n, corr),
                           "roots": n, "depth": d, "A": A, "nodes_per_decision": exp + ev,
                           "parallelism": (f"leaf-range shards x{world}, one NCCL max all-reduce of the "
                                           f"{n * A} packed root keys inside the library") if world > 1
                           else "single GPU",
                           "l2": "flushed before every timed step (256 MiB write, untimed)" if flush is not None
                           else "not flushed", "net_path": "simt" if args.simt else ("tcgen05 tf32" if args.tf32 else "tcgen05")},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step[0] * args.steps,
                "clocks": clk.summary(), "kernels": kernels}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
