#!/usr/bin/env python
"""Benchmark of AMS action-context matching on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c4|c2|c3scan]
                    [--impl ours|reference] [--ungated]
    torchrun --nproc-per-node N ... bench.py --gpus N ...

A step is one ams_match call (query prep -> tcgen05 similarity GEMM with the fused
gate + top-k epilogue -> k-way merge [-> NCCL all-gather -> shard merge]) over the
workload's full query batch against the whole (sharded) pool, inputs resident in HBM.
The default workload is BASELINE.json configs[2] (C3: M=1,048,576, d=1024 bf16, J=14,
Q=16384, k=16, theta 0.9, gamma 0.3), the north_star compute target; the pool is
sharded by rows over N ranks (strong scaling).  Rank 0 prints ONE JSON line.

Extra keys: roofline (dominant kernel, CUDA events on the launching stream; traffic
only from an ncu capture of this very library build), outputs_sha256 (bit-identity
across N), ungated (the same batch with gate_radius = inf), scan (the north_star
64-query HBM-bound scan of the same pool), gate_first_variant (f3), e2e (host buffers
through the C ABI, H2D + D2H inside the timed region), peer_exchange (N > 1: the fused
NVLink exchange of f1, checked bit-identical to the NCCL path), c4 (BASELINE configs[3]
at every N: the 16.8M-row pool resharded over the N ranks, with its own 64-query scan
and output hash), c1 (configs[0], fp32 exact), c2 (configs[1]), c5 (configs[4] streaming, 20 steps),
scaling_sim (N = 1:
per-GPU shard timings of C3 and C4 at 2/4/8 ranks predicting strong scaling), cpu_baseline (the oracle on the host cores, a bounded query sample,
CPU model named), clocks (nvidia-smi during the main timed region; every leg carries its
own window), gpu_launches (our kernels inside the timed region).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "context-match queries/sec and pool-scan HBM GB/s at 1/2/4/8 B200; % roofline"
# The paper never times the lookup itself; its only latency numbers, quoted with their
# hardware as context (not a baseline): the lookup replaces a VLA inference.
PAPER_CONTEXT = {"vla_inference_ms": 200, "action_slice_execution_ms": 1000,
                 "hardware": "GPU not named (pi0 on a JAKA s5 arm)", "source": "PAPER.md:1232 (section 6)",
                 "note": "context only: the paper reports no number for context matching (BASELINE.md)"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm_gbs": p["hbm_gbs"], "bf16_tflops": p["bf16_tflops"],
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained"), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons, sampled every 100 ms from the first timed region
    to the end of the last leg; window(t0, t1) summarises the samples of one leg."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []   # (wall time, fields)
        self.proc = None
        self.th = None
        self.pending = []
        self.stopped = False

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append((time.time(), parts))

    @classmethod
    def summarise(cls, rows):
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        for r in rows:
            for n, v in zip(cls.NAMES, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w_median": statistics.median(pw) if pw else None}

    def _window_rows(self, t0: float, t1: float):
        inside = [r for t, r in self.rows if t0 <= t <= t1 + 0.1]
        if not inside:   # a leg shorter than the sampling period: the first sample after it
            inside = [r for t, r in self.rows if t > t1][:1]
        return inside

    def window(self, t0: float, t1: float):
        """Summary of the samples taken while [t0, t1] ran (at least the first sample after
        it, so a sub-100-ms leg still gets a reading).  Filled in when the sampler stops
        (the returned dict is updated in place), so late samples are not missed."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        out = {"window_s": round(t1 - t0, 4)}
        if self.stopped:
            out.update(self.summarise(self._window_rows(t0, t1)))
        else:
            self.pending.append((t0, t1, out))
        return out

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        self.stopped = True
        for t0, t1, out in self.pending:
            out.update(self.summarise(self._window_rows(t0, t1)))
        self.pending = []
        return self.summarise([r for _, r in self.rows])


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3", choices=["c2", "c3", "c3scan", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ungated", action="store_true", help="gate_radius = +inf")
    ap.add_argument("--no-scan", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="queries in the oracle sample (0 = auto)")
    ap.add_argument("--gate-first", action="store_true",
                    help="time ams_match_gate_first (SURVEY 8(f) f3 variant) instead of the dense ams_match")
    ap.add_argument("--no-variant", action="store_true", help="skip the gate-first side measurement")
    ap.add_argument("--no-ungated", action="store_true", help="skip the ungated (gate_radius = inf) sub-line")
    ap.add_argument("--no-c4", action="store_true", help="skip the configs[3] (C4) block")
    ap.add_argument("--no-c2", action="store_true", help="skip the configs[1] (C2) and configs[0] (C1) blocks")
    ap.add_argument("--no-c5", action="store_true", help="skip the configs[4] (C5 streaming, 20 steps) block")
    ap.add_argument("--no-scaling-sim", action="store_true",
                    help="N = 1 only: skip the per-GPU shard timings that predict 2/4/8-GPU strong scaling")
    ap.add_argument("--no-peer", action="store_true", help="skip the fused peer-exchange side measurement (N > 1)")
    ap.add_argument("--force-collective", action="store_true",
                    help="N = 1 only: run the multi-GPU code path (NCCL all-gather, shard merge, peer exchange) "
                         "over a 1-rank communicator -- a dry run of what --gpus N > 1 executes")
    ap.add_argument("--kernel-policy", type=int, default=0, choices=list(range(16)),
                    help="bit mask for A/B measurements: 1 = batches of <= 128 queries use the 128-query-tile "
                         "kernel instead of the small-batch kernel; 2 = two CTA pairs per 4-CTA cluster sharing "
                         "multicast pool rows (opt-in); 4 = wide small-batch CTA pairs (two tiles per stage, opt-in); 8 = ungated 129-256-query "
                         "batches on the small-batch CTA pairs")
    return ap.parse_args()


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.impl == "ours":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return rank, world, local


def workload_cfg(args):
    import ams_gen
    return ams_gen.CONFIGS[args.workload]


def config_block(cfg, args, world, gamma):
    return {"workload": f"{cfg.name} (BASELINE.json configs[{ {'c1': 0, 'c2': 1, 'c3': 2, 'c3scan': 2, 'c4': 3, 'c5': 4}[cfg.name] }])",
            "M": cfg.M, "d": cfg.d, "J": cfg.J, "Q": cfg.Q, "k": cfg.k, "theta": cfg.theta,
            "gate_radius": gamma, "pool_dtype": cfg.dtype, "shard": f"rows contiguous over {world} rank(s)",
            "l2": "inputs larger than L2 (pool %.2f GB > 126 MB L2)" % (cfg.M * cfg.d * 2 / 1e9),
            "data": "synthetic (ams_gen recipe, DESIGN.md)"}


def oracle_sample(cfg, dev, qn, qjn, gamma, n_s, offset=0):
    """Time the oracle (mode A, all host cores) on n_s of the workload's queries against
    the full pool.  The pool is regenerated chunk by chunk (ams_gen, not timed) and copied
    to the host; the oracle runs per chunk with the chunk's global ids and its
    per-chunk lists are merged by oracle.merge -- exact by pin P8 -- so no host copy of
    the whole pool is needed.  Returns (seconds in the oracle, cores)."""
    import numpy as np
    import torch
    import ams_gen
    import oracle
    sel = (np.arange(n_s) + offset) % qn.shape[0]
    q, qj = np.ascontiguousarray(qn[sel]), np.ascontiguousarray(qjn[sel])
    means = ams_gen.device_means(cfg, dev)
    keys, ids = [], []
    t = 0.0
    nchunks = (cfg.M + ams_gen.CHUNK_ROWS - 1) // ams_gen.CHUNK_ROWS
    group = max(1, (1 << 20) // ams_gen.CHUNK_ROWS)   # ~1M rows per oracle call
    for c0 in range(0, nchunks, group):
        es, js = [], []
        for c in range(c0, min(nchunks, c0 + group)):
            e, j = ams_gen.device_pool_chunk(cfg, c, means, dev)
            es.append(e.view(torch.int16).cpu().numpy().view(np.uint16))
            js.append(j.cpu().numpy())
        e = np.concatenate(es)
        j = np.concatenate(js)
        rid = np.arange(c0 * ams_gen.CHUNK_ROWS, c0 * ams_gen.CHUNK_ROWS + e.shape[0], dtype=np.int64)
        t0 = time.perf_counter()
        r = oracle.match(e, j, q, qj, cfg.k, cfg.theta, gamma, mode="A", row_ids=rid)
        t += time.perf_counter() - t0
        keys.append(r.key)
        ids.append(r.idx)
    t0 = time.perf_counter()
    oracle.merge(np.stack(keys), np.stack(ids), cfg.k, cfg.theta)
    t += time.perf_counter() - t0
    return t, oracle.max_threads()


def auto_sample(cfg, cores):
    # ~1e9 fp64 pair-MACs per core-second: aim for ~20 s of CPU work in total
    per_query = cfg.M * cfg.d / 1e9
    return int(max(1, min(max(cores, 4), round(20.0 / max(per_query, 1e-6)))))


def run_stream(args):
    """C5 (configs[4]) streaming record-and-replay as the bench line (--workload c5)."""
    rank, world, local = dist_setup(args)
    line = stream_measure(args, args.steps, max(args.warmup, 3), rank, world, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as tdist
        tdist.destroy_process_group()


def stream_measure(args, T, W, rank, world, local, route=None):
    """C5 (configs[4]) streaming record-and-replay.  A step = one simulated 20 ms robot
    step: ams_pool_append of 256 new contexts, then the step's 256 queries (50 %
    near-duplicates of rows appended <= 50 steps ago or of initial rows, 50 % mixture)
    in seeded batches of 1..256 (log-uniform).  Every ams_match is timed with CUDA
    events on the launching stream; value = queries/s over the timed steps.  Returns the
    line (rank 0) or None.  route: "dense" | "gate_first" | "auto" (default: --gate-first or
    dense)."""
    import numpy as np
    import torch
    import ams_gen
    import paper_2508_10259_b200 as ams
    from paper_2508_10259_b200 import dist as adist

    cfg = ams_gen.CONFIGS["c5"]
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    route = route or ("gate_first" if args.gate_first else "dense")
    match_fn = {"dense": ams.ams_match, "gate_first": ams.ams_match_gate_first, "auto": ams.ams_match_auto}[route]
    per_step = 256
    cap = cfg.M + per_step * (T + W)
    block = 256
    pool = adist.create_pool(cfg.d, cfg.J, cap, per_step, cfg.k, dtype="bf16", shard_block=block)
    ams.ams_pool_set_kernel_policy(pool.handle, args.kernel_policy)
    dummy = torch.zeros(1, cfg.d, dtype=torch.bfloat16, device=dev)
    dummy_j = torch.zeros(1, cfg.J, dtype=torch.float32, device=dev)

    def append_fn(e, j, n):
        pool.append(dummy, dummy_j, n) if e is None else pool.append(e, j, n)

    need = lambda lo, hi: adist.owned_range_overlaps(cap, world, block, rank, lo, hi)  # noqa: E731
    sup_q, sup_qj, sup_lab = ams_gen.build_device_workload(cfg, dev, append_fn, Q=8192, chunk_needed=need)
    sup_nd = torch.nonzero(sup_lab >= 0).flatten()
    sup_fr = torch.nonzero(sup_lab < 0).flatten()
    # pre-generate every step's rows and queries (generation stays out of the timed region)
    g = torch.Generator(device=dev).manual_seed(cfg.seed * 1_000_003 + 777)
    rows, queries = [], []
    sigma = 0.05 / math.sqrt(cfg.d)
    for s in range(T + W):
        e, j = ams_gen.stream_rows(cfg, s, per_step, dev)
        rows.append((e, j))
        n_nd = per_step // 2
        n_recent = n_nd // 2
        lo = max(0, s - 50)
        src_step = torch.randint(lo, s + 1, (n_recent,), generator=g, device=dev)
        src_row = torch.randint(0, per_step, (n_recent,), generator=g, device=dev)
        re = torch.stack([rows[int(a)][0][int(b)] for a, b in zip(src_step.tolist(), src_row.tolist())]).float()
        rj = torch.stack([rows[int(a)][1][int(b)] for a, b in zip(src_step.tolist(), src_row.tolist())])
        qa = re + sigma * torch.randn(re.shape, generator=g, device=dev)
        qa = qa / torch.linalg.vector_norm(qa, dim=1, keepdim=True)
        qaj = rj + 0.02 * torch.randn(rj.shape, generator=g, device=dev)
        pick_nd = sup_nd[torch.randint(0, sup_nd.numel(), (n_nd - n_recent,), generator=g, device=dev)]
        pick_fr = sup_fr[torch.randint(0, sup_fr.numel(), (per_step - n_nd,), generator=g, device=dev)]
        q = torch.cat([qa.to(torch.bfloat16), sup_q[pick_nd], sup_q[pick_fr]])
        qj = torch.cat([qaj, sup_qj[pick_nd], sup_qj[pick_fr]]).float()
        perm = torch.randperm(per_step, generator=g, device=dev)
        queries.append((q[perm].contiguous(), qj[perm].contiguous(), ams_gen.batch_sizes(per_step, seed=s)))
    torch.cuda.synchronize()
    out_i = torch.empty(per_step, cfg.k, dtype=torch.int64, device=dev)
    out_s = torch.empty(per_step, cfg.k, dtype=torch.float32, device=dev)
    out_h = torch.empty(per_step, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    n_events = sum(len(queries[s][2]) for s in range(W, T + W))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_events)]
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(T)]

    def run_step(s, timed, ev_i):
        e, j = rows[s]
        pool.append(e, j, per_step, stream)
        q, qj, sizes = queries[s]
        off = 0
        for b in sizes:
            if timed:
                evs[ev_i][0].record(stream)
            match_fn(
                pool.handle, q[off:off + b], qj[off:off + b], b, cfg.k, cfg.theta, cfg.gamma, out_i, out_s, out_h,
                stream)
            if timed:
                evs[ev_i][1].record(stream)
                ev_i += 1
            off += b
        return ev_i

    for s in range(W):
        run_step(s, False, 0)
    torch.cuda.synchronize()
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    time.sleep(0.15)
    l0 = ams.ams_pool_launch_count(pool.handle)
    if world > 1:
        import torch.distributed as tdist
        tdist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    ev_i = 0
    for i, s in enumerate(range(W, T + W)):
        step_ev[i][0].record(stream)
        ev_i = run_step(s, True, ev_i)
        step_ev[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    launches = ams.ams_pool_launch_count(pool.handle) - l0
    clocks = clk.stop()
    lat = np.array([a.elapsed_time(b) for a, b in evs])
    bsz = np.array([b for s in range(W, T + W) for b in queries[s][2]])
    by_batch = {name: {"calls": int(m.sum()), "p50": float(np.percentile(lat[m], 50)),
                       "p99": float(np.percentile(lat[m], 99))}
                for name, m in (("nq<=128", bsz <= 128), ("nq>128", bsz > 128)) if m.any()}
    steps_ms = np.array([a.elapsed_time(b) for a, b in step_ev])
    total = t0.elapsed_time(t1)
    if world > 1:
        import torch.distributed as tdist
        tt = torch.tensor([total, float(np.percentile(lat, 50)), float(np.percentile(lat, 99))],
                          dtype=torch.float64, device=dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        total, p50, p99 = tt.tolist()
        tdist.barrier()
    else:
        p50, p99 = float(np.percentile(lat, 50)), float(np.percentile(lat, 99))
    m_now = pool.size
    line = None
    shard_rows = -(-m_now // world)
    bytes_call = shard_rows * (2 * cfg.d + 4 * cfg.J + 4)
    if route == "gate_first":   # the gate-first scan reads the (padded) joints only
        bytes_call = shard_rows * 4 * (4 if cfg.J <= 4 else 8 if cfg.J <= 8 else 16)
    value = per_step * T / (total / 1e3)
    if rank == 0:
        gbs = bytes_call / (np.median(lat) / 1e3) / 1e9
        line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": T, "warmup": W,
                "ms_per_step": total / T, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "c5 (BASELINE.json configs[4]) streaming record-and-replay",
                           "M0": cfg.M, "d": cfg.d, "J": cfg.J, "k": cfg.k, "theta": cfg.theta,
                           "gate_radius": cfg.gamma, "appends_per_step": per_step, "queries_per_step": per_step,
                           "batches": "log-uniform 1..256 (seeded)", "shard": f"block-cyclic 256 over {world} rank(s)",
                           "l2": "inputs larger than L2 (pool %.1f GB)" % (m_now * cfg.d * 2 / 1e9)},
                "latency_ms": {"p50": p50, "p99": p99, "max": float(lat.max()), "calls": int(lat.size),
                               "by_batch_size_rank0": by_batch},
                "step_ms": {"p50": float(np.percentile(steps_ms, 50)), "max": float(steps_ms.max()),
                            "fits_20ms_step": bool(steps_ms.max() < 20.0)},
                "pool_scan_gbps_per_gpu_p50": gbs,
                "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": gbs / peaks["hbm_gbs"], "traffic": None,
                             "note": "whole ams_match call (prep + scan kernel + merge) at the median batch"},
                "clocks": clocks, "gpu_launches": launches, "e2e": None, "cpu_baseline": None,
                "path": {"dense": "ams_match (dense tcgen05)", "gate_first": "ams_match_gate_first",
                         "auto": "ams_match_auto (route per call by sampled pass-rate)"}[route]}
        if route == "auto":
            line["route_last_call"] = ams.ams_pool_last_route(pool.handle)
    pool.close()
    return line


def run_reference(args):
    """The oracle as the reference arm (--impl reference), rank 0 only."""
    import numpy as np
    import torch
    import ams_gen
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cfg = workload_cfg(args)
    gamma = float("inf") if args.ungated else cfg.gamma
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))) if torch.cuda.is_available() else torch.device("cpu")
    noop = lambda e, j, n: None  # noqa: E731
    q, qj, labels = ams_gen.build_device_workload(cfg, dev, noop, chunk_needed=lambda lo, hi: False)
    q = q.view(torch.int16).cpu().numpy().view(np.uint16)
    qj = qj.cpu().numpy()
    cores = oracle.max_threads()
    n_s = args.cpu_sample or max(1, 4 * cores)   # several queries per core: no per-step load imbalance
    per_query_s = cfg.M * cfg.d / 1e9 / max(cores, 1)
    while n_s > 1 and n_s * per_query_s * (args.steps + args.warmup) > 240:
        n_s //= 2
    for w in range(args.warmup):
        oracle_sample(cfg, dev, q, qj, gamma, n_s, offset=w * n_s)
    t = 0.0
    for s in range(args.steps):
        dt, cores = oracle_sample(cfg, dev, q, qj, gamma, n_s, offset=(args.warmup + s) * n_s)
        t += dt
    value = args.steps * n_s / t
    line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_block(cfg, args, 1, gamma),
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"{n_s} queries per step of {cfg.name} against the full pool "
                                       f"({cfg.M} rows), oracle mode A (fp64 brute force, OpenMP over queries) "
                                       f"per ~1M-row chunk + oracle.merge"},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def traffic_of(workload: str, which: str):
    """(dram bytes per launch, source) of the dominant kernel from the committed ncu
    summary -- only if that capture was taken of THIS build (the build id -- a hash of the
    sources, headers and flags compiled into libams.so -- recorded by scripts/ncu_summary.py
    matches the loaded library's ams_build_id()); otherwise (None, why)."""
    import paper_2508_10259_b200 as ams
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            e = json.load(f)[workload][which]
    except Exception:
        return None, "no ncu --set full capture of this kernel/workload in profiles/ncu_summary.json"
    bid = ams.ams_build_id()
    if e.get("build_id") != bid:
        return None, (f"profiles/ncu_summary.json capture ({e.get('round')}, {e.get('report')}) is of another "
                      f"build; not reused")
    return e["dram_bytes_per_launch"], (f"ncu --set full capture {e.get('round')} ({e.get('report')}) of this "
                                        f"build (ams_build_id {bid[:16]}), per launch")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def outputs_sha256(out_i, out_s, out_h) -> str:
    """sha256 of (idx int64, score fp32, hit u8) bytes: bit-identity across N (pin P8 on hardware)."""
    import hashlib
    h = hashlib.sha256()
    for t in (out_i, out_s, out_h):
        h.update(t.contiguous().cpu().numpy().tobytes())
    return h.hexdigest()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "c5":
        run_stream(args)
        return
    import numpy as np
    import torch
    import ams_gen
    import paper_2508_10259_b200 as ams
    from paper_2508_10259_b200 import dist as adist

    rank, world, local = dist_setup(args)
    cfg = workload_cfg(args)
    gamma = float("inf") if args.ungated else cfg.gamma
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    tdist = None
    if world > 1:
        import torch.distributed as tdist
    stream = torch.cuda.current_stream()
    clk = ClockSampler(torch.cuda.current_device())

    def barrier():
        if tdist is not None:
            tdist.barrier()

    def max_over_ranks(x: float) -> float:
        if tdist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def all_ok(ok: bool) -> bool:
        if tdist is None:
            return ok
        t = torch.tensor([0 if ok else 1], dtype=torch.int32, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return int(t.item()) == 0

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def timed(fn, reps):
        """barrier + sync, CUDA events around reps calls on `stream`, sync + barrier;
        (max over ranks of the elapsed ms, wall window for the clock samples)."""
        barrier()
        torch.cuda.synchronize()
        w0 = time.time()
        ev0.record(stream)
        for _ in range(reps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        w1 = time.time()
        barrier()
        return max_over_ranks(ev0.elapsed_time(ev1)), (w0, w1)

    def kernel_avg(pool):
        k_ms, k_n = ams.ams_pool_read_profile(pool.handle)
        return max_over_ranks(k_ms / max(k_n, 1))

    def make_pool(c):
        pool = adist.create_pool(c.d, c.J, c.M, c.Q, c.k, dtype="bf16", shard_block=0,
                                 force_collective=args.force_collective)
        ams.ams_pool_set_kernel_policy(pool.handle, args.kernel_policy)
        dummy = torch.zeros(1, c.d, dtype=torch.bfloat16, device=dev)
        dummy_j = torch.zeros(1, c.J, dtype=torch.float32, device=dev)

        def append_fn(e, j, n):
            if e is None:
                pool.append(dummy, dummy_j, n)   # this rank owns none of these rows
            else:
                pool.append(e, j, n)

        need = lambda lo, hi: adist.owned_range_overlaps(c.M, world, 0, rank, lo, hi)  # noqa: E731
        q, qj, labels = ams_gen.build_device_workload(c, dev, append_fn, chunk_needed=need)
        torch.cuda.synchronize()
        assert pool.size == c.M
        return pool, q, qj, labels

    def shard_sim(c, q, qj, n_shards, reps):
        """Per-GPU step time of an n_shards-way run, predicted on this one GPU: a pool
        holding exactly rank 0's contiguous shard (rows [0, ceil(M/n))) through the world > 1
        code path (1-rank NCCL communicator: shard merge, all-gather, final merge), the full
        query batch.  Excludes only the cross-GPU transfer of the all-gather (G x nq x k x 12
        B, ~3 MB at G = 8 for C3)."""
        m_sh = -(-c.M // n_shards)
        pool_s = adist.create_pool(c.d, c.J, m_sh, c.Q, c.k, dtype="bf16", shard_block=0, force_collective=True)
        ams.ams_pool_set_kernel_policy(pool_s.handle, args.kernel_policy)
        means = ams_gen.device_means(c, dev)
        for ch in range((m_sh + ams_gen.CHUNK_ROWS - 1) // ams_gen.CHUNK_ROWS):
            e, j = ams_gen.device_pool_chunk(c, ch, means, dev)
            n = min(e.shape[0], m_sh - ch * ams_gen.CHUNK_ROWS)
            pool_s.append(e[:n].contiguous(), j[:n].contiguous(), n)
        o = (torch.empty(c.Q, c.k, dtype=torch.int64, device=dev), torch.empty(c.Q, c.k, dtype=torch.float32, device=dev),
             torch.empty(c.Q, dtype=torch.uint8, device=dev))
        fn = lambda: ams.ams_match(pool_s.handle, q, qj, c.Q, c.k, c.theta, c.gamma, *o, stream)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ms, win = timed(fn, reps)
        pool_s.close()
        return ms / reps, clk.window(*win)

    def scaling_sim(c, q, qj, t1_ms, reps):
        out = {"note": "predicted on 1 GPU: per-GPU step time of rank 0's shard through the world > 1 path "
                       "(1-rank NCCL); excludes the cross-GPU all-gather transfer. efficiency = t1 / (N * tN)",
               "t1_ms": t1_ms}
        for n in (2, 4, 8):
            t_n, cl = shard_sim(c, q, qj, n, reps)
            out[f"n{n}"] = {"ms_per_step": t_n, "queries_per_s_per_rank": c.Q / (t_n / 1e3),
                            "predicted_efficiency": t1_ms / (n * t_n), "clocks": cl}
        return out

    def scan_leg(pool, c, q, qj, g, nq=64):
        """The north_star 64-query HBM-bound scan of pool `c` (per GPU shard)."""
        o = (torch.empty(nq, c.k, dtype=torch.int64, device=dev), torch.empty(nq, c.k, dtype=torch.float32, device=dev),
             torch.empty(nq, dtype=torch.uint8, device=dev))
        qs, qjs = q[:nq].contiguous(), qj[:nq].contiguous()
        fn = lambda: ams.ams_match(pool.handle, qs, qjs, nq, c.k, c.theta, g, *o, stream)  # noqa: E731
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        w_ms, _ = timed(fn, 5)
        ams.ams_pool_read_profile(pool.handle)
        ams.ams_pool_set_profiling(pool.handle, True)
        reps = max(20, 5 * args.steps, int(500.0 / max(w_ms / 5, 1e-3)))   # >= ~0.5 s: several clock samples
        ms, win = timed(fn, reps)
        ams.ams_pool_set_profiling(pool.handle, False)
        s_ms = ms / reps
        plan = ams.ams_pool_last_plan(pool.handle)
        k_avg = kernel_avg(pool)
        bytes_shard = (c.M / world) * (2 * c.d + 4 * c.J + 4)
        gbs = bytes_shard / (k_avg / 1e3) / 1e9
        kname = "match_scan" if plan["kernel_id"] == 4 else "match_tc_scan"
        traffic, tsrc = traffic_of(c.name if c.name != "c3scan" else "c3", kname)
        return {"queries": nq, "value": nq / (s_ms / 1e3), "unit": "queries/s", "ms_per_call": s_ms,
                "pool_scan_gbps_per_gpu": bytes_shard / (s_ms / 1e3) / 1e9, "plan": plan,
                "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": gbs / peaks["hbm_gbs"],
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks["source"] == "measured"
                             else "fallback 6650 GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)",
                             "traffic": traffic, "traffic_source": tsrc,
                             "kernel": "match_scan_kernel" if plan["kernel_id"] == 4 else "match_tc_kernel",
                             "kernel_ms_avg": k_avg, "frac_vs_datasheet_8000": gbs / 8000.0,
                             "algorithmic_bytes_per_launch": bytes_shard},
                "clocks": clk.window(*win)}

    # ------------------------------------------------------------------ pool + queries
    pool, q, qj, labels = make_pool(cfg)
    out_i = torch.empty(cfg.Q, cfg.k, dtype=torch.int64, device=dev)
    out_s = torch.empty(cfg.Q, cfg.k, dtype=torch.float32, device=dev)
    out_h = torch.empty(cfg.Q, dtype=torch.uint8, device=dev)
    match_fn = ams.ams_match_gate_first if args.gate_first else ams.ams_match

    def step(qe=q, qjj=qj, nq=cfg.Q, fn=None, g=gamma):
        (fn or match_fn)(pool.handle, qe, qjj, nq, cfg.k, cfg.theta, g, out_i, out_s, out_h, stream)

    # ------------------------------------------------------------------ main timing
    warmups = max(args.warmup, 3)   # the timing rules require >= 3 warm-up steps
    for _ in range(warmups):
        step()
    torch.cuda.synchronize()
    ams.ams_pool_read_profile(pool.handle)            # drop warm-up events
    clk.start()
    time.sleep(0.15)
    ams.ams_pool_set_profiling(pool.handle, True)
    l0 = ams.ams_pool_launch_count(pool.handle)
    t_ms, win_main = timed(step, args.steps)
    launches = ams.ams_pool_launch_count(pool.handle) - l0
    ams.ams_pool_set_profiling(pool.handle, False)
    kern_avg = kernel_avg(pool)
    plan = ams.ams_pool_last_plan(pool.handle)
    hit_rate = float(out_h.float().mean().item())
    out_sha = outputs_sha256(out_i, out_s, out_h)
    lab = labels.cpu().numpy()
    top1 = out_i[:, 0].cpu().numpy()
    nd = lab >= 0
    label_top1 = float(np.mean(top1[nd] == lab[nd])) if nd.any() else None

    value = cfg.Q * args.steps / (t_ms / 1e3)
    m_shard = -(-cfg.M // world)
    flops_launch = 2.0 * cfg.Q * m_shard * cfg.d
    bytes_step = cfg.M * (2 * cfg.d + 4 * cfg.J + 4)
    achieved_tf = flops_launch / (kern_avg / 1e3) / 1e12
    traffic, tsrc = traffic_of(args.workload, "match_tc")
    roofline = {"bound": "tensor", "achieved": achieved_tf, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": achieved_tf / peaks["bf16_tflops"], "traffic": traffic, "traffic_source": tsrc,
                "kernel": "match_tc_kernel (tcgen05 GEMM + fused gate/top-k epilogue)",
                "algorithmic_per_launch": {"flop": flops_launch, "bytes": bytes_step / world},
                "kernel_ms_avg": kern_avg, "kernel_share_of_step": kern_avg / (t_ms / args.steps),
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if peaks["source"] == "measured"
                else "fallback 1590 TF burst (B200_PROFILING.md; MEASURED_PEAKS.json absent)",
                "frac_vs_sustained": achieved_tf / peaks["bf16_tflops_sustained"]
                if peaks.get("bf16_tflops_sustained") else None,
                "frac_vs_datasheet_2250": achieved_tf / 2250.0}

    if not args.gate_first and cfg.Q <= 128:   # below the ridge (~250 flop/B): HBM-bound scan
        gbs = (bytes_step / world) / (kern_avg / 1e3) / 1e9
        kname = "match_scan" if plan.get("kernel_id") == 4 else "match_tc"
        traffic, tsrc = traffic_of(args.workload, kname)
        roofline = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / peaks["hbm_gbs"], "traffic": traffic, "traffic_source": tsrc,
                    "kernel": "match_scan_kernel" if plan.get("kernel_id") == 4 else "match_tc_kernel",
                    "algorithmic_per_launch": {"bytes": bytes_step / world, "flop": flops_launch},
                    "kernel_ms_avg": kern_avg, "kernel_share_of_step": kern_avg / (t_ms / args.steps),
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks["source"] == "measured"
                    else "fallback 6650 GB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"}

    if args.gate_first:   # the dominant kernels read only joints: report against HBM
        jp = 4 if cfg.J <= 4 else 8 if cfg.J <= 8 else 16
        jbytes = m_shard * 4 * jp
        gbs = jbytes / (kern_avg / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": gbs / peaks["hbm_gbs"], "traffic": None, "traffic_source": "not captured",
                    "kernel": "gate_scan_kernel + score_kernel (gate-first variant)",
                    "algorithmic_per_launch": {"bytes": jbytes}, "kernel_ms_avg": kern_avg,
                    "note": "joint bytes per launch / kernel time; the scan is ALU-bound, so this is low by design"}

    # ------------------------------------------------------------------ ungated sub-line
    ungated = None
    if not args.no_ungated and not args.gate_first and math.isfinite(gamma) and cfg.Q > 128:
        g_inf = float("inf")
        step(g=g_inf)
        torch.cuda.synchronize()
        ams.ams_pool_read_profile(pool.handle)
        ams.ams_pool_set_profiling(pool.handle, True)
        u_ms, win = timed(lambda: step(g=g_inf), args.steps)
        ams.ams_pool_set_profiling(pool.handle, False)
        u_k = kernel_avg(pool)
        u_tf = flops_launch / (u_k / 1e3) / 1e12
        ungated = {"gate_radius": "inf", "value": cfg.Q * args.steps / (u_ms / 1e3), "unit": "queries/s",
                   "ms_per_step": u_ms / args.steps, "kernel_ms_avg": u_k, "achieved_tflops": u_tf,
                   "frac": u_tf / peaks["bf16_tflops"], "outputs_sha256": outputs_sha256(out_i, out_s, out_h),
                   "clocks": clk.window(*win)}

    # ------------------------------------------------------------------ 64-query scan
    scan = None
    if not args.no_scan and cfg.Q >= 64:
        scan = scan_leg(pool, cfg, q, qj, gamma)

    # ------------------------------------------------------------------ gate-first variant (f3)
    variant = None
    if not args.no_variant and not args.gate_first and math.isfinite(gamma):
        res = {}
        for label, nq in (("full_batch", cfg.Q), ("scan_64", min(64, cfg.Q))):
            qv, qjv = q[:nq].contiguous(), qj[:nq].contiguous()
            for _ in range(3):
                step(qv, qjv, nq, ams.ams_match_gate_first)
            torch.cuda.synchronize()
            reps = max(5, args.steps)
            v_ms, win = timed(lambda: step(qv, qjv, nq, ams.ams_match_gate_first), reps)
            v_ms /= reps
            res[label] = {"queries": nq, "ms_per_call": v_ms, "value": nq / (v_ms / 1e3), "unit": "queries/s",
                          "joint_bytes_gbps_per_gpu": (cfg.M / world) * 4 * (8 if cfg.J <= 8 else 16) / (v_ms / 1e3) / 1e9,
                          "clocks": clk.window(*win)}
        variant = {"name": "ams_match_gate_first (SURVEY 8(f) f3; exact, gate evaluated first)", **res}

    # ------------------------------------------------------------------ route selection (f3 auto)
    auto = None
    if not args.no_variant and not args.gate_first:
        res = {}
        for label, nq in (("full_batch", cfg.Q), ("scan_64", min(64, cfg.Q))):
            qv, qjv = q[:nq].contiguous(), qj[:nq].contiguous()
            for _ in range(3):
                step(qv, qjv, nq, ams.ams_match_auto)
            torch.cuda.synchronize()
            reps = max(5, args.steps)
            a_ms, win = timed(lambda: step(qv, qjv, nq, ams.ams_match_auto), reps)
            r = ams.ams_pool_last_route(pool.handle)
            m_loc = cfg.M / world
            res[label] = {"queries": nq, "ms_per_call": a_ms / reps, "value": nq / (a_ms / reps / 1e3),
                          "unit": "queries/s", "route": r["route"],
                          "est_eligible_rows_per_query": r["est_eligible_per_query"],
                          "est_pass_rate": (r["est_eligible_per_query"] / m_loc) if r["est_eligible_per_query"] >= 0
                          else None, "cost_model_ms": {"dense": r["est_ms_dense"], "gate_first": r["est_ms_gate_first"]},
                          "clocks": clk.window(*win)}
        auto = {"name": "ams_match_auto (SURVEY 8(f) f3: route by sampled pass-rate + cost model)", **res}

    # ------------------------------------------------------------------ e2e (host buffers)
    e2e = None
    if not args.no_e2e:
        hq = q.cpu().pin_memory()
        hqj = qj.cpu().pin_memory()
        ho_i = torch.empty(cfg.Q, cfg.k, dtype=torch.int64).pin_memory()
        ho_s = torch.empty(cfg.Q, cfg.k, dtype=torch.float32).pin_memory()
        ho_h = torch.empty(cfg.Q, dtype=torch.uint8).pin_memory()

        def e2e_step():
            ams.ams_match(pool.handle, hq, hqj, cfg.Q, cfg.k, cfg.theta, gamma, out_i, out_s, out_h, stream)
            ho_i.copy_(out_i, non_blocking=True)
            ho_s.copy_(out_s, non_blocking=True)
            ho_h.copy_(out_h, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e_ms, win = timed(e2e_step, args.steps)
        h2d = hq.numel() * hq.element_size() + hqj.numel() * hqj.element_size()
        d2h = ho_i.numel() * 8 + ho_s.numel() * 4 + ho_h.numel()
        e2e = {"value": cfg.Q * args.steps / (e_ms / 1e3), "unit": "queries/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "path": "ams_match(host pinned q, q_joints) + D2H of idx/score/hit",
               "clocks": clk.window(*win)}

    # ------------------------------------------------------------------ fused peer exchange (f1), N > 1
    peer = None
    if (world > 1 or args.force_collective) and not args.no_peer and not args.gate_first:
        try:
            ams.ams_pool_enable_peer_exchange(pool.handle)
            ok, why = True, ""
        except Exception as e:   # collective inside the library: every rank gets the same status
            ok, why = False, str(e)
        if all_ok(ok):
            try:
                step()
                torch.cuda.synchronize()
                same = outputs_sha256(out_i, out_s, out_h) == out_sha
                p_ms, win = timed(step, args.steps)
                st = ams.ams_pool_status(pool.handle)
                same = same and outputs_sha256(out_i, out_s, out_h) == out_sha
                peer = {"status": "ok" if st == 0 else ams.ams_status_string(st),
                        "value": cfg.Q * args.steps / (p_ms / 1e3), "unit": "queries/s",
                        "ms_per_step": p_ms / args.steps, "bit_identical_to_nccl_path": bool(all_ok(same)),
                        "clocks": clk.window(*win)}
            except Exception as e:
                peer = {"status": "error", "error": str(e)}
        else:
            peer = {"status": "unsupported", "error": why or "a peer rank could not map the exchange buffers"}

    # ------------------------------------------------------------------ CPU oracle baseline
    cpu = None
    want_cpu = (not args.no_cpu_baseline) and world == 1 and rank == 0
    if want_cpu:
        qn = q.view(torch.int16).cpu().numpy().view(np.uint16)
        qjn = qj.cpu().numpy()
        import oracle
        cores = oracle.max_threads()
        n_s = args.cpu_sample or auto_sample(cfg, cores)
        dt, cores = oracle_sample(cfg, dev, qn, qjn, gamma, n_s)
        if not args.cpu_sample and dt < 8.0 and n_s < cfg.Q:
            # calibrated: rescale the sample to ~15 s of oracle time (contract: 10-30 s)
            n_s = int(min(cfg.Q, max(n_s + 1, round(n_s * 15.0 / max(dt, 1e-3)))))
            dt, cores = oracle_sample(cfg, dev, qn, qjn, gamma, n_s)
        cpu = {"value": n_s / dt, "unit": "queries/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"first {n_s} of the {cfg.Q} {cfg.name} queries against the full {cfg.M}-row pool, "
                         f"oracle mode A (fp64 brute force, OpenMP over queries) per ~1M-row chunk + oracle.merge, "
                         f"{dt:.1f} s in the oracle"}
    pool.close()
    sim3 = None
    if world == 1 and args.workload == "c3" and not args.no_scaling_sim and not args.gate_first:
        sim3 = scaling_sim(cfg, q, qj, t_ms / args.steps, args.steps)
    del q, qj

    # ------------------------------------------------------------------ C4 (configs[3]) at every N
    c4 = None
    if args.workload == "c3" and not args.no_c4:
        c4cfg = ams_gen.CONFIGS["c4"]
        pool4, q4, qj4, _ = make_pool(c4cfg)
        o4 = (torch.empty(c4cfg.Q, c4cfg.k, dtype=torch.int64, device=dev),
              torch.empty(c4cfg.Q, c4cfg.k, dtype=torch.float32, device=dev),
              torch.empty(c4cfg.Q, dtype=torch.uint8, device=dev))
        fn4 = lambda: ams.ams_match(pool4.handle, q4, qj4, c4cfg.Q, c4cfg.k, c4cfg.theta, c4cfg.gamma, *o4,  # noqa: E731
                                    stream)
        for _ in range(3):
            fn4()
        torch.cuda.synchronize()
        ams.ams_pool_read_profile(pool4.handle)
        ams.ams_pool_set_profiling(pool4.handle, True)
        reps4 = max(3, args.steps // 4)
        c_ms, win = timed(fn4, reps4)
        ams.ams_pool_set_profiling(pool4.handle, False)
        k4 = kernel_avg(pool4)
        fl4 = 2.0 * c4cfg.Q * (-(-c4cfg.M // world)) * c4cfg.d
        tf4 = fl4 / (k4 / 1e3) / 1e12
        c4 = {"workload": "c4 (BASELINE.json configs[3]): M=16,777,216 d=1024 bf16 J=7, Q=8192, k=32, theta 0.9, "
                          f"gamma 0.3; rows contiguous over {world} rank(s)",
              "value": c4cfg.Q * reps4 / (c_ms / 1e3), "unit": "queries/s", "n_gpus": world, "steps": reps4,
              "warmup": 3, "ms_per_step": c_ms / reps4, "scaling": "strong",
              "roofline": {"bound": "tensor", "achieved": tf4, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                           "frac": tf4 / peaks["bf16_tflops"], "kernel_ms_avg": k4,
                           "algorithmic_per_launch": {"flop": fl4}},
              "plan": ams.ams_pool_last_plan(pool4.handle), "outputs_sha256": outputs_sha256(*o4),
              "clocks": clk.window(*win)}
        if not args.no_scan:
            c4["scan"] = scan_leg(pool4, c4cfg, q4, qj4, c4cfg.gamma)
        pool4.close()
        if world == 1 and not args.no_scaling_sim:
            c4["scaling_sim"] = scaling_sim(c4cfg, q4, qj4, c_ms / reps4, reps4)
    # ------------------------------------------------------------------ C2 (configs[1]) at every N
    c2 = None
    if args.workload == "c3" and not args.no_c2:
        c2cfg = ams_gen.CONFIGS["c2"]
        w2 = ams_gen.generate_host(c2cfg)
        pool2 = adist.create_pool(c2cfg.d, c2cfg.J, c2cfg.M, c2cfg.Q, c2cfg.k, dtype="bf16", shard_block=0,
                                  force_collective=args.force_collective)
        pool2.append(w2.emb, w2.joints, c2cfg.M)
        q2 = torch.from_numpy(w2.q_emb).to(dev).view(torch.bfloat16)
        qj2 = torch.from_numpy(w2.q_joints).to(dev)
        o2 = (torch.empty(c2cfg.Q, c2cfg.k, dtype=torch.int64, device=dev),
              torch.empty(c2cfg.Q, c2cfg.k, dtype=torch.float32, device=dev),
              torch.empty(c2cfg.Q, dtype=torch.uint8, device=dev))
        fn2 = lambda: ams.ams_match(pool2.handle, q2, qj2, c2cfg.Q, c2cfg.k, c2cfg.theta, c2cfg.gamma, *o2,  # noqa: E731
                                    stream)
        for _ in range(5):
            fn2()
        torch.cuda.synchronize()
        ams.ams_pool_read_profile(pool2.handle)
        ams.ams_pool_set_profiling(pool2.handle, True)
        reps2 = max(50, 5 * args.steps)
        c_ms, win = timed(fn2, reps2)
        ams.ams_pool_set_profiling(pool2.handle, False)
        k2 = kernel_avg(pool2)
        fl2 = 2.0 * c2cfg.Q * (-(-c2cfg.M // world)) * c2cfg.d
        nd2 = w2.labels >= 0
        c2 = {"workload": "c2 (BASELINE.json configs[1]): M=100,000 d=768 bf16 J=7, Q=4096, k=10, theta 0.92, "
                          f"gamma 0.3; rows contiguous over {world} rank(s)",
              "value": c2cfg.Q * reps2 / (c_ms / 1e3), "unit": "queries/s", "steps": reps2, "warmup": 5,
              "ms_per_step": c_ms / reps2,
              "roofline": {"bound": "tensor", "achieved": fl2 / (k2 / 1e3) / 1e12, "peak": peaks["bf16_tflops"],
                           "unit": "TFLOP/s", "frac": fl2 / (k2 / 1e3) / 1e12 / peaks["bf16_tflops"],
                           "kernel_ms_avg": k2},
              "hits_equal_near_duplicates": bool(np.array_equal(o2[2].cpu().numpy().astype(bool), nd2)),
              "outputs_sha256": outputs_sha256(*o2), "clocks": clk.window(*win)}
        pool2.close()

    # ------------------------------------------------------------------ C1 (configs[0]) fp32 exact, every N
    c1 = None
    if args.workload == "c3" and not args.no_c2:
        c1cfg = ams_gen.CONFIGS["c1"]
        w1 = ams_gen.generate_host(c1cfg)
        pool1 = adist.create_pool(c1cfg.d, c1cfg.J, c1cfg.M, c1cfg.Q, c1cfg.k, dtype="fp32", shard_block=0,
                                  force_collective=args.force_collective)
        pool1.append(w1.emb, w1.joints, c1cfg.M)
        q1 = torch.from_numpy(w1.q_emb).to(dev)
        qj1 = torch.from_numpy(w1.q_joints).to(dev)
        o1 = (torch.empty(c1cfg.Q, c1cfg.k, dtype=torch.int64, device=dev),
              torch.empty(c1cfg.Q, c1cfg.k, dtype=torch.float32, device=dev),
              torch.empty(c1cfg.Q, dtype=torch.uint8, device=dev))
        fn1 = lambda: ams.ams_match(pool1.handle, q1, qj1, c1cfg.Q, c1cfg.k, c1cfg.theta, c1cfg.gamma, *o1,  # noqa: E731
                                    stream)
        for _ in range(10):
            fn1()
        torch.cuda.synchronize()
        reps1 = 2000
        m1, win = timed(fn1, reps1)
        nd1 = w1.labels >= 0
        c1 = {"workload": "c1 (BASELINE.json configs[0]): M=1024 d=512 fp32 J=7, Q=64, k=5, theta 0.9, gamma 0.3 "
                          "(the bit-exact canonical fp32 path; launch/latency-bound)",
              "value": c1cfg.Q * reps1 / (m1 / 1e3), "unit": "queries/s", "us_per_call": 1e3 * m1 / reps1,
              "steps": reps1, "plan": ams.ams_pool_last_plan(pool1.handle),
              "hits_equal_near_duplicates": bool(np.array_equal(o1[2].cpu().numpy().astype(bool), nd1)),
              "top1_equals_source": bool(np.array_equal(o1[0][:, 0].cpu().numpy()[nd1], w1.labels[nd1])),
              "outputs_sha256": outputs_sha256(*o1), "clocks": clk.window(*win)}
        pool1.close()

    # ------------------------------------------------------------------ C5 (configs[4]) streaming
    c5 = None
    if args.workload == "c3" and not args.no_c5:
        w0 = time.time()
        c5l = stream_measure(args, 20, 3, rank, world, local)
        if c5l is not None:
            c5 = {k: c5l[k] for k in ("value", "unit", "ms_per_step", "latency_ms", "step_ms",
                                      "pool_scan_gbps_per_gpu_p50", "roofline", "clocks", "gpu_launches")}
            c5["workload"] = c5l["config"]["workload"] + f", {c5l['steps']} timed steps after {c5l['warmup']} warm-up"
            c5["shard"] = c5l["config"]["shard"]
            c5["wall_s"] = round(time.time() - w0, 1)
        # the same loop through ams_match_auto (f3 route selection): the robot-step budget
        c5a = stream_measure(args, 20, 3, rank, world, local, route="auto")
        if c5a is not None and c5 is not None:
            c5["auto_route"] = {k: c5a[k] for k in ("value", "latency_ms", "step_ms", "route_last_call", "clocks")}

    clocks_all = clk.stop()
    clocks = clk.window(*win_main)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
                "warmup": warmups, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": config_block(cfg, args, world, gamma),
                "pool_scan_gbps_per_gpu": (bytes_step / world) / (t_ms / args.steps / 1e3) / 1e9,
                "collective_path": bool(world > 1 or args.force_collective),
                "roofline": roofline, "outputs_sha256": out_sha, "ungated": ungated, "scan": scan,
                "gate_first_variant": variant, "auto_route": auto, "e2e": e2e, "peer_exchange": peer, "c4": c4,
                "c1": c1, "c2": c2, "c5": c5, "scaling_sim": sim3, "cpu_baseline": cpu,
                "clocks": clocks, "clocks_whole_run": clocks_all,
                "gpu_launches": launches, "plan": plan, "hit_rate": hit_rate, "path": "ams_match_gate_first"
                if args.gate_first else "ams_match (dense tcgen05)",
                "near_dup_top1_equals_source": label_top1,
                "paper_context": PAPER_CONTEXT}
        print(json.dumps(line), flush=True)
    if tdist is not None:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
