#!/usr/bin/env python
"""Benchmark of the STree tree-verify hot path (BASELINE.json metric:
"tree-verify nodes/s per SSM layer (1/2/4/8 B200); % of roofline").

One STEP = one verify iteration of an L-layer Mamba-2 stack over one batch of
synthetic drafted trees, i.e. one pass through every §8(a) row, in Alg. 1's
order (ActivationReplay, TreeScan, FirstRejected):
    stree_build_mask (once) -> L x stree_replay_scan (commit of the previous
    step's accepted path into the layer state + scan of the tree) -> stree_accept
With --no-fuse the commit runs as separate kernels after accept:
    stree_build_mask -> L x stree_tree_scan -> stree_accept -> L x stree_commit
Workload (default) = BASELINE configs[3] / SURVEY c4 per GPU: 16 random
recursive trees x 64 nodes, Mamba-2 2.7B layer shape (H=80, P=64, N=128, G=1),
bf16 x/B/C/y, fp32 dt/A/D/state, L = 64 distinct layers (every layer has its
own buffers, 4.1 GB in total, > 30x the 126 MB L2, so no L2 flush is needed).

value = B*T*L*world / max-over-ranks(step time)  [nodes/s per layer, whole job].
Each phase of the step (mask / scans / accept / commits) is one CUDA graph;
CUDA events between the graph launches on the launching stream give the
per-kernel average durations used in the roofline object.

--impl reference runs the CPU oracle (oracle/, fp64) as the reference arm on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from gen import inputs  # noqa: E402

METRIC = "tree-verify nodes/s per SSM layer"
UNIT = "nodes/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="stree", choices=["stree", "reference"])
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4"])
    ap.add_argument("--layers", type=int, default=64)
    ap.add_argument("--scan-impl", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-early-state", action="store_true")
    ap.add_argument("--no-fuse", action="store_true",
                    help="separate commit kernels instead of the fused replay+scan (stree_replay_scan)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next", action="store_true",
                    help="skip the SURVEY §8(f) rows (tree attention, KV commit, tree conv, conv commit; bench_next.py)")
    ap.add_argument("--p-match", type=float, default=0.9)
    ap.add_argument("--shard", default="heads", choices=["batch", "heads"],
                    help="N>1: heads (default, BASELINE configs[3]) = ranks split the heads of the same 16 trees, "
                         "the scan epilogue writes every y tile into every rank's full-y buffer over NVLink "
                         "(symmetric memory; NCCL all-gather if unavailable), strong scaling; batch = each rank "
                         "verifies its own trees (no collective, weak scaling)")
    ap.add_argument("--no-p2p", action="store_true", help="heads: NCCL all-gather instead of epilogue P2P stores")
    ap.add_argument("--force-heads", action="store_true",
                    help="run the head-sharded code path (symmetric memory, sharded scan, barrier) even at N=1")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(cfg, prob, L):
    d = prob.dims
    return {"workload": f"{cfg}: Mamba-2 2.7B-shaped SSM layer stack, tree verify "
                        f"(mask, scan + commit of {L} layers, accept)" if cfg != "c2" else
            f"{cfg}: Mamba-2 130M-shaped layer stack, tree verify",
            "trees_per_gpu": d.batch, "nodes_per_tree": d.n_nodes, "heads": d.n_heads, "head_dim": d.head_dim,
            "d_state": d.d_state, "n_groups": d.n_groups, "layers": L, "io_dtype": d.io_dtype,
            "state_dtype": "f32", "tree": "random recursive, branching<=4" if cfg == "c4" else "heap binary",
            "l2": "inputs larger than L2 (distinct per-layer buffers, no reuse within a step)"}


def scan_bytes(d):
    s_io = 2 if d.io_dtype == "bf16" else 4
    B, T, H, P, N, G = d.batch, d.n_nodes, d.n_heads, d.head_dim, d.d_state, d.n_groups
    return B * (T * H * P * (s_io + s_io) + T * H * 4 + 2 * T * G * N * s_io + H * P * N * 4 + T * 4) + H * 8


def commit_bytes(d, path_len):
    s_io = 2 if d.io_dtype == "bf16" else 4
    H, P, N = d.n_heads, d.head_dim, d.d_state
    return int(sum(2 * H * P * N * 4 + int(r) * (H * P * s_io + H * 4 + N * s_io) for r in path_len))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def load_traffic(cfg):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            j = json.load(f)
        out = dict(j.get(cfg) or {})
        out["_source"] = j.get("source", "profiles/traffic.json")
        return out
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi-equivalent sampling through NVML during the timed region."""

    def __init__(self, index, period=0.01):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
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
        nv = self.nv
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU oracle timing (reference arm / cpu_baseline)
# ---------------------------------------------------------------------------
def oracle_sample(prob, tok, vt, n_trees):
    """One bounded oracle 'step' on the first n_trees trees of one layer:
    mask + scan + accept + commit (fp64, OpenMP over (tree, head))."""
    import oracle
    sl = slice(0, n_trees)
    x, Bm, Cm = prob.io_as_f32("x")[sl], prob.io_as_f32("Bm")[sl], prob.io_as_f32("Cm")[sl]
    par = prob.parent[sl]
    t0 = time.perf_counter()
    oracle.build_mask(par)
    oracle.tree_scan(x, prob.dt[sl], prob.A, Bm, Cm, prob.D, prob.h0[sl], par)
    path, plen, _, _ = oracle.accept(tok[sl], par, vt[sl])
    oracle.commit(x, prob.dt[sl], prob.A, Bm, prob.h0[sl], path, plen, par)
    return time.perf_counter() - t0


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    prob = inputs.config_problem(args.config)
    tok, vt = inputs.make_accept_inputs(prob.parent, seed=123, p_match=args.p_match)
    n_trees = 1
    # calibrate the sample: grow until one step takes >= ~2 s (bounded by the batch)
    dt_ = oracle_sample(prob, tok, vt, n_trees)
    while dt_ < 2.0 and n_trees < prob.dims.batch:
        n_trees = min(prob.dims.batch, n_trees * 2)
        dt_ = oracle_sample(prob, tok, vt, n_trees)
    for _ in range(args.warmup):
        oracle_sample(prob, tok, vt, n_trees)
    times = [oracle_sample(prob, tok, vt, n_trees) for _ in range(args.steps)]
    t = sum(times) / len(times)
    value = n_trees * prob.dims.n_nodes / t
    cores = oracle.num_threads()
    sample = (f"{n_trees} of {prob.dims.batch} trees x 1 layer per step (mask+scan+accept+commit), "
              f"fp64 C oracle, OpenMP {cores} threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_desc(args.config, prob, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def cpu_baseline(prob, tok, vt, budget_s=15.0):
    import oracle
    n = 1
    t = oracle_sample(prob, tok, vt, n)
    while t * 2 < 4.0 and n < prob.dims.batch:
        n = min(prob.dims.batch, n * 2)
        t = oracle_sample(prob, tok, vt, n)
    reps, tot = 0, 0.0
    while tot < budget_s and reps < 20:
        tot += oracle_sample(prob, tok, vt, n)
        reps += 1
    cores = oracle.num_threads()
    out = {"value": n * prob.dims.n_nodes * reps / tot, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{n} trees x 1 layer (mask+scan+accept+commit) x {reps} reps of {args_cfg_name(prob)}, "
                     f"fp64, {tot:.1f} s, OpenMP {cores} threads",
           "cpu_model": oracle.cpu_model(), "build": "gcc -O3 -march=native -ffp-contract=off -fopenmp"}
    # the same oracle on one thread: one tree per sample, ~1/3 of the budget
    oracle.set_threads(1)
    try:
        reps1, tot1 = 0, 0.0
        while tot1 < budget_s / 3 and reps1 < 20:
            tot1 += oracle_sample(prob, tok, vt, 1)
            reps1 += 1
    finally:
        oracle.set_threads(0)
    out["single_thread"] = {"value": prob.dims.n_nodes * reps1 / tot1, "unit": UNIT, "cores": 1,
                            "sample": f"1 tree x 1 layer x {reps1} reps, {tot1:.1f} s"}
    return out


def args_cfg_name(prob):
    d = prob.dims
    return f"B={d.batch} T={d.n_nodes} H={d.n_heads} P={d.head_dim} N={d.d_state}"


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_stree(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2505_14969_b200 import api, binding

    binding.stree_set_scan_impl({"auto": 0, "simt": 1, "tc": 2}[args.scan_impl])
    # PDL between consecutive kernels; in this step the kernel preceding a scan / commit of layer l never
    # writes layer l's state, so the state stream may start before the dependency wait (EARLY_STATE)
    binding.stree_set_launch_flags(binding.STREE_LAUNCH_PDL |
                                   (0 if args.no_early_state else
                                    binding.STREE_LAUNCH_EARLY_STATE | binding.STREE_LAUNCH_EARLY_REPLAY |
                                    binding.STREE_LAUNCH_EARLY_TREE | binding.STREE_LAUNCH_EARLY_DT))
    L = args.layers
    base0 = inputs.config_problem(args.config)
    # distinct per-layer buffers must exceed the 126 MB L2 (no flush needed): small layers get more of them
    lb = scan_bytes(base0.dims) + base0.dims.batch * base0.dims.n_heads * base0.dims.head_dim * base0.dims.d_state * 4
    if args.layers == 64 and lb * L < 2 * 126e6:
        L = int(-(-2 * 126e6 // lb))
    # every rank verifies its own batch of trees (weak scaling; no data-path collective)
    from paper_2505_14969_b200 import dist as sdist
    base = inputs.config_problem(args.config)
    d = base.dims
    par_np = base.parent
    heads_mode = (world > 1 and args.shard == "heads") or args.force_heads
    if args.force_heads and not dist.is_initialized():   # one-rank group for the symmetric-memory rendezvous
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    h_lo, h_hi = sdist.shard_heads(d.n_heads, d.n_groups, world, rank) if heads_mode else (0, d.n_heads)
    if world > 1 and not heads_mode:
        rng = np.random.default_rng(inputs.BASE_SEED + 1000 + rank)
        from gen import trees as _t
        par_np = np.stack([_t.random_recursive(d.n_nodes, 4, rng) for _ in range(d.batch)]) \
            if args.config == "c4" else par_np
    H_full = d.n_heads
    if heads_mode:
        import dataclasses
        d = dataclasses.replace(d, n_heads=h_hi - h_lo, n_groups=max(1, d.n_groups * (h_hi - h_lo) // d.n_heads))
    seed_rank = 0 if heads_mode else rank
    tok, vt = inputs.make_accept_inputs(par_np, seed=inputs.BASE_SEED + 77 + seed_rank, p_match=args.p_match)

    # per-layer inputs: distinct buffers (values generated on device to keep setup fast;
    # layer 0 is the seeded host problem, the others are seeded device randoms of the same recipe)
    g = torch.Generator(device=dev)
    g.manual_seed(inputs.BASE_SEED + 10 * rank)
    layers = []
    t0 = api.upload(inputs.make_problem(d, par_np, seed=inputs.BASE_SEED + 3 + 100 * rank), device=dev)
    ygath = None
    io_t = t0["x"].dtype
    for li in range(L):
        if li == 0:
            t = t0
        else:
            B, T, H, P, N, G = d.batch, d.n_nodes, d.n_heads, d.head_dim, d.d_state, d.n_groups
            t = {
                "x": torch.randn((B, T, H, P), generator=g, device=dev).to(io_t),
                "dt": torch.exp(torch.empty((B, T, H), device=dev).uniform_(np.log(1e-3), np.log(1e-1),
                                                                            generator=g)),
                "A": -torch.empty((H,), device=dev).uniform_(1.0, 16.0, generator=g),
                "Bm": torch.randn((B, T, G, N), generator=g, device=dev).to(io_t),
                "Cm": torch.randn((B, T, G, N), generator=g, device=dev).to(io_t),
                "D": 1 + 0.1 * torch.randn((H,), generator=g, device=dev),
                "h0": torch.randn((B, H, P, N), generator=g, device=dev),
                "parent": t0["parent"],
            }
        t["y"] = torch.empty_like(t["x"])
        layers.append(t)
    parent = t0["parent"]
    tok_d = torch.from_numpy(tok).to(dev)
    vt_d = torch.from_numpy(vt).to(dev)
    W = (d.n_nodes + 31) // 32
    mask = torch.empty((d.batch, d.n_nodes, W), dtype=torch.int32, device=dev)
    depth = torch.empty((d.batch, d.n_nodes), dtype=torch.int32, device=dev)
    path = torch.empty((d.batch, d.n_nodes), dtype=torch.int32, device=dev)
    plen = torch.empty((d.batch,), dtype=torch.int32, device=dev)
    bonus = torch.empty((d.batch,), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    dims = binding.make_dims(layers[0]["x"], layers[0]["Bm"])
    kernel = binding.stree_scan_kernel_for(dims)

    def ph_mask():
        binding.stree_build_mask(parent, mask, depth, status)

    def ph_scan():
        for t in layers:
            binding.stree_tree_scan(t["x"], t["dt"], t["A"], t["Bm"], t["Cm"], t["D"], t["h0"], parent, t["y"],
                                    status, dims=dims)

    def ph_accept():
        binding.stree_accept(tok_d, parent, vt_d, path, plen, bonus, status)

    # head-sharded layer: the full y of every layer on every rank (BASELINE configs[3])
    fully, youts = None, None
    if heads_mode:
        fully = sdist.FullY(L, d.batch, d.n_nodes, H_full, d.head_dim, io_t, dev, prefer_p2p=not args.no_p2p,
                            force_p2p=args.force_heads)
        if fully.mode == "p2p":
            youts = [binding.make_yout(fully.peers(li), H_full, h_lo) for li in range(L)]
        if rank == 0:
            print(f"[bench] heads x{world}: full y via {fully.mode}" +
                  (f" (symmetric memory unavailable: {fully.error})" if fully.error else ""), file=sys.stderr)

    def ph_replay_scan():
        # commit of the previous step's accepted path (cache = this layer's x, dt, B of that step)
        # fused with the scan of the current tree, state updated in place; head-sharded + P2P: the epilogue
        # stores every y tile into every rank's full y
        for li, t in enumerate(layers):
            if youts is not None:
                binding.stree_replay_scan_sharded(t["x"], t["dt"], t["Bm"], parent, path, plen, t["x"], t["dt"],
                                                  t["A"], t["Bm"], t["Cm"], t["D"], t["h0"], parent, youts[li],
                                                  status, dims_prev=dims, dims=dims)
            else:
                binding.stree_replay_scan(t["x"], t["dt"], t["Bm"], parent, path, plen, t["x"], t["dt"], t["A"],
                                          t["Bm"], t["Cm"], t["D"], t["h0"], parent, t["y"], status,
                                          dims_prev=dims, dims=dims)

    def ph_collect():
        # heads: make the full y of every layer visible on every rank (P2P: the device barrier that publishes
        # the epilogue stores; NCCL: all-gather of the local shards)
        if fully.mode == "p2p":
            fully.publish()
        else:
            for li, t in enumerate(layers):
                fully.gather(li, t["y"])

    def ph_commit():
        for t in layers:
            binding.stree_commit(t["x"], t["dt"], t["A"], t["Bm"], t["h0"], parent, path, plen, t["h0"], status,
                                 dims=dims)

    fused = not args.no_fuse
    phases = [ph_mask, ph_replay_scan, ph_accept] if fused else [ph_mask, ph_scan, ph_accept, ph_commit]
    if heads_mode:
        phases.insert(2, ph_collect)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        ph_mask()
        ph_scan()
        ph_accept()        # a valid accepted path exists before the first replay
        for f in phases:   # eager warm-up (loads modules, sets smem attributes)
            f()
    torch.cuda.synchronize()
    graphs = []
    for f in phases:
        try:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                f()
            graphs.append(gr)
        except Exception as exc:   # e.g. a collective that cannot be captured: replay eagerly
            if rank == 0:
                print(f"[bench] graph capture failed ({exc}); running phase eagerly", file=sys.stderr)
            graphs.append(f)
    torch.cuda.synchronize()
    assert status.item() == 0, f"device status {status.item()}"
    plen_host = plen.cpu().numpy()

    def step(evs=None):
        for i, gr in enumerate(graphs):
            if evs is not None:
                evs[i].record(stream)
            if callable(gr):
                gr()
            else:
                gr.replay()
        if evs is not None:
            evs[len(graphs)].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(graphs) + 1)] for _ in range(K)]
    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    with sampler:
        with torch.cuda.stream(stream):
            for k in range(K):
                step(evs[k])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    phase_ms = np.array([[evs[k][i].elapsed_time(evs[k][i + 1]) for i in range(len(graphs))] for k in range(K)])
    total_ms = float(evs[0][0].elapsed_time(evs[K - 1][len(graphs)]))
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / K
    nodes_per_step = d.batch * d.n_nodes * L * (1 if heads_mode else world)
    value = nodes_per_step / (ms_per_step * 1e-3)
    ph_mean = phase_ms.mean(0)
    ph = dict(zip([f.__name__ for f in phases], ph_mean))   # ms per phase
    hbm_peak, bf16_peak, peak_src = load_peaks()
    sb = scan_bytes(d)
    cb = commit_bytes(d, plen_host)
    traffic = load_traffic(args.config) or {}
    kernels = {"stree_build_mask": {"us": ph["ph_mask"] * 1e3}, "stree_accept": {"us": ph["ph_accept"] * 1e3}}
    if heads_mode:
        kernels["collective"] = {"us_per_step": ph["ph_collect"] * 1e3, "mode": fully.mode,
                                 "y_bytes_per_rank_per_layer": fully.layer_bytes,
                                 "note": "p2p: the scan epilogue already stored every y tile into every rank's "
                                         "full y (inside stree_replay_scan_sharded); this is the publishing barrier"
                                 if fully.mode == "p2p" else "NCCL all_gather of the head shards + layout"}
    if fused:
        # fused bytes: the scan's bytes + the committed state written back + the previous path's rows
        fb = sb + cb - d.batch * d.n_heads * d.head_dim * d.d_state * 4
        fu_us = ph["ph_replay_scan"] * 1e3 / L
        fu_gbs = fb / (fu_us * 1e-6) / 1e9
        kernels["stree_replay_scan"] = {"us": fu_us, "bytes": fb, "GB/s": fu_gbs, "frac": fu_gbs / hbm_peak,
                                        "impl": {1: "simt+commit", 2: "tcgen05 fused", 4: "tcgen05 small-batch fused"}.get(kernel),
                                        "mean_path_len": float(plen_host.mean())}
        dominant, dom_gbs, dom_bytes = "stree_replay_scan", fu_gbs, fb
    else:
        scan_us = ph["ph_scan"] * 1e3 / L
        commit_us = ph["ph_commit"] * 1e3 / L
        scan_gbs = sb / (scan_us * 1e-6) / 1e9
        commit_gbs = cb / (commit_us * 1e-6) / 1e9
        kernels["stree_tree_scan"] = {"us": scan_us, "bytes": sb, "GB/s": scan_gbs, "frac": scan_gbs / hbm_peak,
                                      "impl": {1: "simt", 2: "tcgen05", 3: "tcgen05 128-row", 4: "tcgen05 small-batch"}.get(kernel)}
        kernels["stree_commit"] = {"us": commit_us, "bytes": cb, "GB/s": commit_gbs, "frac": commit_gbs / hbm_peak,
                                   "impl": {1: "ring (CUDA cores)", 2: "TMA pipeline"}.get(
                                       binding.stree_commit_kernel_for(dims, True)),
                                   "mean_path_len": float(plen_host.mean())}
        dominant = "stree_tree_scan" if scan_us >= commit_us else "stree_commit"
        dom_gbs, dom_bytes = (scan_gbs, sb) if dominant == "stree_tree_scan" else (commit_gbs, cb)
    # one isolated call of the dominant kernel (launch included, GPU idle before it, no PDL overlap): the
    # latency a single verify step of one layer sees, next to the amortised per-layer time of the graph
    iso = isolated_call_us(phases[1], layers, stream, L)
    kernels[dominant]["isolated_call_us"] = iso
    roofline = {"bound": "hbm", "kernel": dominant, "achieved": dom_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": dom_gbs / hbm_peak, "traffic": traffic.get(dominant), "peak_source": peak_src,
                "traffic_source": traffic.get("_source", "profiles/traffic.json"),
                "algorithmic_bytes_per_launch": dom_bytes, "kernels": kernels}

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, layers, parent, tok_d, vt_d, path, plen, bonus, status, dims, stream, world, dev, d, L,
                      fused, fully, youts)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if heads_mode else "weak",
            "vs_baseline": None,
            "dtype": d.io_dtype, "data": "synthetic", "config": workload_desc(args.config, base, L),
            "gpu_launches": ((L + 2) if fused else (2 * L + 2)) * K, "roofline": roofline, "e2e": e2e,
            "step": "mask + L x replay_scan (fused commit+scan) + accept" if fused else
                    "mask + L x scan + accept + L x commit",
            "clocks": sampler.summary(),
            "parallelism": (f"heads x{world} (full y: {fully.mode})" if heads_mode else
                            f"batch-replicas x{world}") if world > 1 else "single"}
    if world == 1 and not args.no_next:
        # §8(f) rows measured beside the step (their own graphs, after the timed region)
        import bench_next
        line["next_rows"] = bench_next.measure(dev, hbm_peak, bf16_peak)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(base, tok, vt)
    if rank == 0:
        emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def isolated_call_us(phase, layers, stream, L, reps=15):
    """Median over `reps` trials of ONE layer's call of the phase's kernel on its own: device time from the
    event after a ~25 us spin kernel (which keeps the host launch overhead out of the interval) to the
    kernel's completion — the kernel's full latency including its launch boundary, no PDL overlap."""
    import torch
    one = layers[:1]
    saved = list(layers)
    times = []
    try:
        layers[:] = one
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                torch.cuda._sleep(50000)
                e0.record(stream)
                phase()
                e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3)
    finally:
        layers[:] = saved
    return float(statistics.median(times))


def run_e2e(args, layers, parent, tok_d, vt_d, path, plen, bonus, status, dims, stream, world, dev, d, L, fused,
            fully=None, youts=None):
    """Same step through the public API, inputs copied from pinned host memory
    every step (x, dt, B, C of every layer + tree + tokens) and the acceptance
    result (path, path_len, bonus) read back."""
    import torch
    import torch.distributed as dist
    from paper_2505_14969_b200 import binding

    # each layer's inputs (x, dt, B, C) live in ONE pinned host block and ONE device block (256-byte aligned views),
    # so a layer is one host->device copy (many small copies cost more per byte on PCIe than one large one)
    keys = ("x", "dt", "Bm", "Cm")

    def layout(t):
        offs, o = {}, 0
        for k in keys:
            offs[k] = o
            o += -(-t[k].numel() * t[k].element_size() // 256) * 256
        return offs, o

    def views(block, t, offs):
        return {k: block[offs[k]:offs[k] + t[k].numel() * t[k].element_size()].view(t[k].dtype).view(t[k].shape)
                for k in keys}

    host, hblk, dblk = [], [], [[]]
    for t in layers:
        offs, nbytes = layout(t)
        hb = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        hv = views(hb, t, offs)
        for k in keys:
            hv[k].copy_(t[k].cpu())
        host.append(hv)
        hblk.append(hb)
        db = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        dv = views(db, t, offs)
        for k in keys:
            dv[k].copy_(t[k])
        dblk[0].append((db, dv))
    # the verified tree's x, dt, B are the cache the next step's replay reads, so the
    # fused loop double-buffers them: step k uploads into set k % 2 and replays from set (k - 1) % 2
    bufs = [[dv for _, dv in dblk[0]]]
    if fused:
        dblk.append([])
        for t in layers:
            offs, nbytes = layout(t)
            db = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            dv = views(db, t, offs)
            for k in keys:
                dv[k].copy_(t[k])
            dblk[1].append((db, dv))
        bufs.append([dv for _, dv in dblk[1]])
    it = [0]
    hp = parent.cpu().pin_memory()
    htok, hvt = tok_d.cpu().pin_memory(), vt_d.cpu().pin_memory()
    out = [torch.empty(path.shape, dtype=torch.int32).pin_memory(),
           torch.empty(plen.shape, dtype=torch.int32).pin_memory(),
           torch.empty(bonus.shape, dtype=torch.int32).pin_memory()]
    h2d = sum(hb.numel() for hb in hblk) + (hp.numel() + htok.numel() + hvt.numel()) * 4   # incl. alignment padding
    d2h = sum(o.numel() * 4 for o in out)

    # host->device copies run on their own stream, layer by layer, so layer l's kernel overlaps the copy
    # of layer l+1 (PCIe bound: the step time is ~ the copy time of the whole step's inputs)
    cstream = torch.cuda.Stream(device=dev)
    evs = [torch.cuda.Event() for _ in range(len(layers) + 1)]

    def step():
        cur = bufs[it[0] % len(bufs)]
        prv = bufs[(it[0] - 1) % len(bufs)]
        it[0] += 1
        cstream.wait_stream(stream)   # previous step's kernels are done with the buffers
        with torch.cuda.stream(cstream):
            parent.copy_(hp, non_blocking=True)
            tok_d.copy_(htok, non_blocking=True)
            vt_d.copy_(hvt, non_blocking=True)
            evs[-1].record(cstream)
            cb = dblk[(it[0] - 1) % len(dblk)]
            for (db, _), hb, ev in zip(cb, hblk, evs):
                db.copy_(hb, non_blocking=True)   # the layer's x, dt, B, C in one transfer
                ev.record(cstream)
        with torch.cuda.stream(stream):
            stream.wait_event(evs[-1])
            binding.stree_build_mask(parent, torch.empty((d.batch, d.n_nodes, (d.n_nodes + 31) // 32),
                                                         dtype=torch.int32, device=dev), None, status)
            for li, (t, c, p, ev) in enumerate(zip(layers, cur, prv, evs)):
                stream.wait_event(ev)
                if fused and youts is not None:   # head-sharded, epilogue P2P stores into every rank's full y
                    binding.stree_replay_scan_sharded(p["x"], p["dt"], p["Bm"], parent, path, plen, c["x"], c["dt"],
                                                      t["A"], c["Bm"], c["Cm"], t["D"], t["h0"], parent, youts[li],
                                                      status, dims_prev=dims, dims=dims)
                elif fused:   # (the tree topology is the same every step here, so parent serves both trees)
                    binding.stree_replay_scan(p["x"], p["dt"], p["Bm"], parent, path, plen, c["x"], c["dt"], t["A"],
                                              c["Bm"], c["Cm"], t["D"], t["h0"], parent, t["y"], status,
                                              dims_prev=dims, dims=dims)
                else:
                    binding.stree_tree_scan(c["x"], c["dt"], t["A"], c["Bm"], c["Cm"], t["D"], t["h0"], parent,
                                            t["y"], status, dims=dims)
            if fully is not None:   # heads: the full y of every layer on every rank
                if fully.mode == "p2p":
                    fully.publish()
                else:
                    for li, t in enumerate(layers):
                        fully.gather(li, t["y"])
            binding.stree_accept(tok_d, parent, vt_d, path, plen, bonus, status)
            if not fused:
                for t, c in zip(layers, cur):
                    binding.stree_commit(c["x"], c["dt"], t["A"], c["Bm"], t["h0"], parent, path, plen, t["h0"],
                                         status, dims=dims)
            for o, s in zip(out, (path, plen, bonus)):
                o.copy_(s, non_blocking=True)
        stream.synchronize()

    for _ in range(2):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    K = max(3, args.steps // 3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return {"value": d.batch * d.n_nodes * L * (1 if fully is not None else world) / (ms * 1e-3), "unit": UNIT,
            "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": K}


_JSON_FD = None   # the real stdout, reserved for the one JSON line (see main)


def emit(line):
    """Write the bench line to the real stdout: libraries (NCCL prints its version banner on rank 0, torch
    warnings) write to fd 1 too, so main() points fd 1 at stderr and keeps the original for this line only."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_stree(args)


if __name__ == "__main__":
    sys.exit(main())
