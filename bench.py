"""Benchmark: maximal bicliques/s of the B200 MBEA path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: one rank per GPU, NCCL)

A step = one full enumeration of the config's graph (every level-1 subtree,
split over the ranks), with the graph resident in HBM.  Between timed steps a
256 MiB buffer is written to flush L2 (the graph is L2-sized).  Times are CUDA
events on the launch stream, max over ranks.  `e2e` repeats the step through
the public C ABI from host buffers (load with H2D copies -> enumerate -> D2H
result -> free).  `--impl reference` times the CPU oracle (oracle/, plain
Algorithm 1) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "maximal bicliques/sec"
UNIT = "bicliques/s"
MASK64 = (1 << 64) - 1
WORKLOADS = {
    "C1": "C1a crown K12,12 minus a perfect matching (4094 bicliques)",
    "C1b": "C1b G(200,200,0.05), seed 0x2401050390000001",
    "C2": "C2 synthetic power-law bipartite 94,238 x 30,087, 293,360 edges (YouTube-membership-shaped)",
    "C3": "C3 synthetic power-law bipartite 56,519 x 120,867, 440,237 edges (GitHub-shaped)",
    "C4": "C4 synthetic power-law bipartite 105,278 x 340,523, 1,149,739 edges (BookCrossing-shaped)",
    "C5": "C5 synthetic power-law bipartite 545,195 x 96,678, 1,301,942 edges (StackOverflow-shaped)",
}


def graph_of(name):
    from paper_2401_05039_b200 import inputs as I

    return I.crown(12) if name == "C1" else I.config_graph(name)


# ------------------------------------------------------------------ distributed helpers (also unit-tested on gloo)
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def limbs_of(count: int, h: int):
    """(count, hash) -> 8 int64 limbs of 16 bits, so a sum over <= 2^47 ranks cannot overflow."""
    out = []
    for v in (count & MASK64, h & MASK64):
        out += [(v >> (16 * k)) & 0xFFFF for k in range(4)]
    return out


def from_limbs(limbs):
    vals = []
    for j in range(2):
        v = 0
        for k in range(4):
            v += int(limbs[4 * j + k]) << (16 * k)
        vals.append(v & MASK64)
    return vals[0], vals[1]


def allreduce_result(count, h, device, group=None):
    """Sum (count, hash mod 2^64) over ranks: the only data collective of the path (NCCL)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(limbs_of(count, h), dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return from_limbs(t.tolist())


def max_over_ranks(x: float, device) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def wait_ready(self, timeout: float = 3.0):
        """nvidia-smi's start-up (NVML init) must not overlap the timed steps: wait for its first sample."""
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)

    def window(self, t0: float, t1: float):
        """Keep only the samples taken inside the timed region [t0, t1] (all of them if none fall inside)."""
        self.t_window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = list(self.lines)
        if getattr(self, "t_window", None):
            inside = [x for x in lines if self.t_window[0] <= x[0] <= self.t_window[1]]
            lines = inside or lines
        for _, line in lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle (cpu_baseline / reference arm)
def oracle_rate(g, target_s: float, seed: int = 7, config: str = ""):
    """Oracle bicliques/s on a bounded sample of level-1 subtrees.

    Per-root oracle cost is extremely heavy-tailed: on C2/C5 the heaviest 1% of roots (by 2-hop
    size) hold ~90-95% of the oracle's work and single roots take minutes, so no small sample that
    includes them has a bounded time.  The sample therefore EXCLUDES the heaviest 1% and takes every
    k-th remaining root in cost order, as ONE oracle call (k calibrated by a pilot to ~target_s).
    This flatters the CPU (several-fold); the recorded full-run oracle time is reported beside it.
    """
    import oracle

    side = 2 if g.n2 < g.n1 else 1
    n = g.n1 if side == 1 else g.n2
    threads = os.cpu_count() or 1
    e = g.edges().astype(np.int64)
    cand, other = (e[:, 0], e[:, 1]) if side == 1 else (e[:, 1], e[:, 0])
    deg_other = np.bincount(other, minlength=g.n2 if side == 1 else g.n1)
    proxy = np.bincount(cand, weights=deg_other[other], minlength=n)
    order = np.argsort(proxy, kind="stable").astype(np.uint32)[: max(1, int(n * 0.99))]

    def run(k):
        roots = order[(seed % k)::k]
        t0 = time.perf_counter()
        pr = oracle.mbea_roots(g, roots, candidate_side=side)
        return int(pr[:, 0].sum()), time.perf_counter() - t0, len(roots)

    k = max(1, len(order) // 400)
    cnt, dt, m = run(k)
    for _ in range(3):
        if dt >= 0.5 * target_s or k == 1:
            break
        k = max(1, int(k * dt / target_s))
        cnt, dt, m = run(k)
    return cnt / dt, dict(count=cnt, seconds=dt, roots=m, frac=m / n, threads=threads, side=side, k=k)


def golden_full_run(config):
    """The oracle's full-run time for this config, as recorded by scripts/make_golden.py (context)."""
    p = os.path.join(ROOT, "tests", "golden", "configs.txt")
    if os.path.exists(p):
        for line in open(p):
            f = line.split()
            if f and f[0] == config and len(f) >= 7:
                secs, thr = float(f[5]), int(f[6])
                return {"bicliques_per_s": int(f[1]) / secs, "seconds": secs, "threads": thr,
                        "source": "tests/golden/configs.txt (scripts/make_golden.py, all level-1 subtrees)"}
    return None


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle

    oracle.build_oracle()
    g = graph_of(args.config)
    per_step_target = max(3.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    rates, infos = [], []
    for s in range(args.warmup + args.steps):
        r, info = oracle_rate(g, per_step_target, seed=7 + s, config=args.config)
        if s >= args.warmup:
            rates.append(r)
            infos.append(info)
    value = float(np.mean(rates))
    info = infos[-1]
    sample = (f"{info['roots']} of the level-1 subtrees ({100 * info['frac']:.2f}%: every {info['k']}-th root in 2-hop-size "
              f"order, heaviest 1% excluded), {info['count']} bicliques in {info['seconds']:.1f} s per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean([i["seconds"] for i in infos])),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOADS.get(args.config, args.config), "parallelism": "CPU threads over level-1 subtrees"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["threads"], "kind": "oracle", "sample": sample,
                         "full_run": golden_full_run(args.config)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config):
    """dram bytes per launch of the search kernel from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(config)
        if d and d.get("dram_bytes_per_launch") is not None:
            return float(d["dram_bytes_per_launch"])
    return None


def load_ncu(config):
    """Issue / SIMT / cache figures of the search kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get(config)
    if not d:
        return None
    m = d.get("metrics", {})

    def num(k):
        try:
            return float(str(m[k]).split()[0])
        except (KeyError, ValueError, IndexError):
            return None

    dur = d.get("duration_ms_under_ncu")
    dram = d.get("dram_bytes_per_launch")
    lane = num("smsp__thread_inst_executed_per_inst_executed.ratio")
    return {"source": f"profiles/{d.get('name', config)}.md (one serialised launch under ncu)",
            "dram_gbs": dram / dur / 1e6 if dram and dur else None,
            "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "simt_lane_efficiency": lane / 32.0 if lane else None,
            "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
            "top_stalls_pct": dict(list(d.get("stall_pct", {}).items())[:3])}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2401_05039_b200 import MBE_STATS, MBEGraph, mbe_enumerate, mbe_free, mbe_get_info, mbe_load_csr
    from paper_2401_05039_b200 import make_config

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    g = graph_of(args.config)
    stream = torch.cuda.current_stream(dev)
    knobs = dict(ctas_per_sm=args.ctas, threads_per_cta=args.threads, bitmap_threshold=args.T)
    G = MBEGraph.from_graph(g, device=local)

    # one untimed stats pass: algorithmic bytes of this rank's share (deterministic search tree)
    st = G.enumerate(flags=MBE_STATS, rank=rank, world=world, stream=stream.cuda_stream, **knobs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        r = G.enumerate(rank=rank, world=world, stream=stream.cuda_stream, **knobs)
        if world > 1:
            c, h = allreduce_result(r.count, r.hash, dev)
        else:
            c, h = r.count, r.hash
        return r, c, h

    times, kms, results = [], [], []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.wait_ready()
        for _ in range(args.warmup):
            flush.zero_()
            step()
        t_timed = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            ev0.record(stream)
            r, c, h = step()
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            ms = ev0.elapsed_time(ev1)
            times.append(max_over_ranks(ms, dev) if world > 1 else ms)
            kms.append(max_over_ranks(r.kernel_ms, dev) if world > 1 else r.kernel_ms)
            results.append((c, h))
        clk.window(t_timed, time.perf_counter() + 0.15)
    assert all(x == results[0] for x in results), "result changed between steps"
    count, h = results[0]
    ms_per_step = float(np.mean(times))
    step_ms = [round(t, 3) for t in times]
    value = count / (ms_per_step / 1e3)

    # e2e through the public C ABI from host buffers: load (H2D) -> enumerate -> D2H result -> free
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.uint64)
    ci = np.ascontiguousarray(g.col_idx, dtype=np.uint32)
    rp_pin = torch.from_numpy(rp).pin_memory().numpy()
    ci_pin = torch.from_numpy(ci).pin_memory().numpy()
    e2e_t, h2d = [], 0
    for k in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        hd = mbe_load_csr(g.n1, g.n2, rp_pin, ci_pin, device=local)
        r = mbe_enumerate(hd, make_config(rank=rank, world=world, stream=stream.cuda_stream, **knobs))
        info = mbe_get_info(hd)
        mbe_free(hd)
        if world > 1:
            allreduce_result(r.count, r.hash, dev)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            e2e_t.append(max_over_ranks(dt, dev) if world > 1 else dt)
            h2d = int(info["h2d_bytes"])
    e2e_value = count / float(np.mean(e2e_t))

    # roofline of the dominant kernel (the persistent search kernel)
    alg_bytes = st.alg_bytes
    kernel_ms = float(np.mean(kms))
    if world > 1:
        t = torch.tensor([alg_bytes], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        alg_bytes = float(t.item())
    peak, peak_src = load_peaks()
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    traffic = load_traffic(args.config) if world == 1 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle

        oracle.build_oracle()
        rate, info = oracle_rate(g, args.cpu_seconds, config=args.config)
        full = golden_full_run(args.config)
        cpu = {"value": rate, "unit": UNIT, "cores": info["threads"], "kind": "oracle", "full_run": full,
               "sample": f"{info['roots']} level-1 subtrees ({100 * info['frac']:.2f}%: every {info['k']}-th root in "
                         f"2-hop-size order, heaviest 1% excluded, one oracle call), {info['count']} bicliques in {info['seconds']:.1f} s"}
    if rank == 0:
        total_warps = st.n_warps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "count": count, "hash": f"{h:#018x}",
                       "candidate_side": st.candidate_side, "warps_per_gpu": total_warps,
                       "l2": "256 MiB buffer written between timed steps (graph fits in L2)",
                       "parallelism": f"level-1 subtrees dealt over {world} rank(s); intra-GPU warp work stealing",
                       "kernel_ms": kernel_ms, "step_ms": step_ms},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 184, "ms_per_step": 1e3 * float(np.mean(e2e_t))},
            "gpu_launches": 2 * args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "alg_bytes_per_launch": alg_bytes, "kernel": "mbe_search_kernel"},
            "ncu": load_ncu(args.config) if world == 1 else None,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "stats": {"tasks": st.tasks, "pruned": st.pruned, "list_tasks": st.list_tasks,
                      "bitmap_tasks": st.bitmap_tasks, "frames": st.frames, "max_depth": st.max_depth,
                      "phase_frac": [round(c / max(1, st.n_warps * st.kernel_ms * 1.965e6), 4)
                                     for c in st.phase_cycles[:15]]},
        }
        print(json.dumps(line), flush=True)
    G.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    # BASELINE.json: the metric is "8xB200 vs 1 GPU vs CPU oracle" and configs[4] (C5) is the config
    # it names for 1/2/4/8-GPU scaling, so C5 is the default workload; C2..C4 via --config.
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
