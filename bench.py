#!/usr/bin/env python3
"""bench.py -- configurations evaluated per second by the ParaDL sweep on 1..8 B200.

Headline workload (BASELINE.json configs[4], the largest sweep that is
also the 8-GPU target): ResNet-152 pipeline + data parallelism -- every contiguous partition of
the 152 rows into s <= 6 stages (633,245,832 partitions) x S in {1,2,4,8} x p_d in 2^0..2^7 x
a 2 x 2 alpha/beta grid = 81,055,466,496 configurations per step.  A step is one pass of the
hot path over the whole sweep: decode -> Table 2 cost -> feasibility -> top-64 / argmin /
feasible count, per rank over its tile shard, then (N > 1) one NCCL all_gather of the
per-rank top-k records and the device merge.  N > 1 defaults to strong scaling (the fixed
sweep split N ways); `--scaling weak` crosses the sweep with N FLOP rates instead and is
reported under a different metric name.  `value` = configurations / s for the whole job
(inputs resident: model + spec image loaded before the timed region); `e2e` = the same
through the public C-ABI with host inputs and host results (paradl_set_system +
paradl_topk each step, which re-uploads the spec image and reads back the hits).
`configs` = the other BASELINE configs (1-4) timed the same way, one line each.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5]
Under torchrun (N > 1) each rank drives LOCAL_RANK's GPU; rank 0 prints one JSON line.
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
sys.path.insert(0, ROOT)

K_TOP = 64
METRIC = "oracle configs evaluated/sec at 1/2/4/8 B200; % of FP64 issue roofline"
METRIC_WEAK = METRIC + " [weak scaling: the sweep crossed with N FLOP rates, N x the configurations]"
# Algorithmic FP64-pipe instructions per configuration: the alpha/beta-dependent increment of
# the canonical tree after hoisting what is invariant over the inner radices
# (s*beta is formed once per beta slot, alpha-side products once per alpha row and shared by
# the M = n_beta/32 slots: 1/M each, M = 2 in the bench sweeps).  Pipeline family:
# (alpha + s*beta), c*( ), comp + ( ), *I = 4.  The top-k admission test is an integer
# compare of the key's high word (not FP64) and is not counted.
M_SLOTS = 2.0
FP64_OPS_PER_CONFIG = {"pipeline": 4.0, "data": 4.0, "filter": 6.0 + 1 / M_SLOTS, "channel": 6.0 + 1 / M_SLOTS,
                       "spatial": 7.0 + 1 / M_SLOTS, "df": 9.0 + 1 / M_SLOTS, "ds": 10.0 + 1 / M_SLOTS,
                       "pd": 7.0, "layerpure": 4.0 + 1 / M_SLOTS, "serial": 1.0,
                       "spatial_ag": 10.0 + 1 / M_SLOTS,
                       # per-layer strategy (Q39): per alpha row 2 (n alpha products), per
                       # configuration GE 3, Allgather 2, changes 2, ag 1, t folds 2, AR 1, key 1
                       "layerwise": 14.0}


def fp64_per_config(sb) -> float:
    """Algorithmic FP64 instructions per feasible configuration of a sub-sweep.
    Pipeline / pd sub-sweeps with a small alpha x beta block run the lane-blocked screened
    nest: per configuration t = comp + G, t += P (pd; pipeline has no G), with G = ge_c (alpha
    + ge_s beta) shared by the 4 S values of a pass and P = pp_c (alpha + pp_s beta) shared by
    the dims values; the admission screen is an integer min of t's high word and one key = t * I
    per pass (the key is monotone in t)."""
    from workloads import sweeps as W
    fam = W.FAMILY_NAMES[sb.family]
    nab = max(1, len(sb.alpha)) * max(1, len(sb.beta))
    if fam == "pipeline" and sb.part_mode == W.PART_MASK and nab * max(1, len(sb.S)) * max(1, len(sb.dims)) == 1:
        # one configuration per mask (cfg3-ii): every configuration is its own structure. The
        # canonical tree per mask, with what is invariant per stage count (cseg, pp_c, alpha,
        # beta) and per table entry (U tau, bS D(delta Y) beta: a maximum of monotone products
        # is the product of the maximum) hoisted exactly: D(maxF + maxB), x cseg, x tau,
        # + U tau, alpha + Yb, x pp_c, comp + P2P = 7; x I once per 512-mask block on the
        # smallest t_iter (the key is monotone in t_iter; DESIGN.md §5.1 mask blocks)
        return 7.0 + 1.0 / 512
    if fam in ("pd", "pipeline") and nab < 32:
        n_s, n_d = max(1, len(sb.S)), max(1, len(sb.dims))
        g = 3.0 * math.ceil(n_s / 4) / n_s if fam == "pd" else 0.0
        key = math.ceil(n_s / 4) / (n_s * nab)   # x I once per pass of 4 S x 4 alpha/beta rows
        return (2.0 if fam == "pd" else 1.0) + key + g + 3.0 / n_d
    return float(FP64_OPS_PER_CONFIG[fam])


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target oracle time for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the SURVEY §8(f) next-row sweeps")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = the fixed sweep split N ways (default, the headline metric); weak = "
                         "the sweep crossed with N per-GPU FLOP rates (N x the configurations, each rank's shard "
                         "the size of the 1-GPU sweep), reported under a separate metric name")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config lines for the other BASELINE configs")
    return ap.parse_args()


def bench_sweep(args, ws: int):
    """The timed sweep.  N = 1: BASELINE config `args.config` as is.  N > 1 with weak scaling:
    every sub-sweep crossed with N FLOP rates R0 (1 + r/4), r = 0..N-1 (the paper's system-
    parameter radix, P:706 'all the permutations of possible configurations'); slice r = 0 is
    the 1-GPU sweep, and the per-rank top-k are merged over NCCL as in strong scaling."""
    from workloads import sweeps as W
    base_sweep = W.CONFIGS[args.config]()
    if args.scaling == "weak" and ws > 1:
        R0 = base_sweep.system.flops_per_s
        for sb in base_sweep.subs:
            base = list(sb.flops) or [R0]
            sb.flops = [f * (1.0 + 0.25 * r) for r in range(ws) for f in base]
        base_sweep.name = f"{base_sweep.name}_x{ws}_flops"
    return base_sweep


# ------------------------------------------------------------------ clocks (nvidia-smi)
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names[1:], parts[5:9]):
                if v.lower() in ("active", "0x1", "1", "yes"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ distributed plumbing
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model() -> str:
    """Host CPU model name (lscpu 'Model name', else /proc/cpuinfo)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def golden_check(cfg: int, sweep, n: int, hits, n_feasible: int):
    """Compares a whole-sweep top-k with the oracle golden tests/golden/full_cfgN.json (written
    offline by tools/golden_full.py from oracle/ alone; a stored file, the oracle is not run).
    None when no golden exists for this workload."""
    path = os.path.join(ROOT, "tests", "golden", f"full_cfg{cfg}.json")
    if not os.path.exists(path):
        return None
    g = json.load(open(path))
    if g.get("workload") != sweep.name or g.get("configs") != n:
        return None
    gh = [(i, float.fromhex(k)) for i, k in g["hits"]]
    ours = [(int(i), float(k)) for i, k in hits[:len(gh)]]
    return {"golden": os.path.relpath(path, ROOT), "topk_identical": ours == gh,
            "count_identical": int(n_feasible) == int(g["n_feasible"]), "k": len(gh)}


def cpu_oracle_baseline(sweep, target_s: float, rank: int = 0):
    """The oracle as it stands, on all host cores, on a bounded sample of the same sweep:
    contiguous windows of 4096 configurations at evenly spaced offsets."""
    from oracle import oracle as O
    osw = O.OracleSweep(sweep)
    n = osw.size()
    cores = os.cpu_count() or 1

    def run(nwin):
        stride = n // nwin
        t0 = time.perf_counter()
        tot = 0
        for w in range(nwin):
            a = w * stride
            c = min(4096, n - a)
            osw.topk(a, c, K_TOP, nthreads=cores)
            tot += c
        return tot, time.perf_counter() - t0

    tot, dt = run(8)
    nwin = max(8, int(8 * target_s / max(dt, 1e-3)))
    tot, dt = run(nwin)
    return {"value": tot / dt, "unit": "configs/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{nwin} windows x 4096 consecutive configs evenly spaced over the {n}-config sweep "
                      f"({tot} configs, {dt:.1f} s, top-{K_TOP} + count per window)"}


def bench_config(sweep, n_configs: int, ws: int) -> dict:
    """The `config` object of both arms (same keys and values for the same workload)."""
    return {"workload": sweep.name, "configs_per_step": int(n_configs), "k": K_TOP,
            "model": "+".join(m.name for m in sweep.models) + " layer tables (paper Table 4 shapes)",
            "parallelism": f"index-range shards x{ws} + NCCL all_gather merge",
            "l2": "flushed (256 MiB device write) before every timed step; inputs are a KB-size image"}


def reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from workloads import sweeps as W
    sweep = bench_sweep(args, dist_env()[0])
    base = {"metric": METRIC if args.scaling == "strong" or args.gpus <= 1 else METRIC_WEAK,
            "unit": "configs/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": None}
    per_step_s = max(0.3, min(5.0, 120.0 / max(1, args.steps + args.warmup)))
    from oracle import oracle as O
    osw = O.OracleSweep(sweep)
    n = osw.size()
    base["config"] = bench_config(sweep, n, dist_env()[0])
    cores = os.cpu_count() or 1
    # calibrate windows per step so one step takes about per_step_s seconds
    t0 = time.perf_counter()
    osw.topk(0, 4096, K_TOP, nthreads=cores)
    dt1 = time.perf_counter() - t0
    nwin = max(1, int(per_step_s / max(dt1, 1e-4)))
    stride = max(1, n // nwin)
    times = []
    tot = 0
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for w in range(nwin):
            a = (w * stride + s * 4096) % max(1, n - 4096)
            osw.topk(a, 4096, K_TOP, nthreads=cores)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            tot += nwin * 4096
    v = tot / sum(times)
    line = dict(base, value=v, ms_per_step=1e3 * sum(times) / len(times),
                cpu_baseline={"value": v, "unit": "configs/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                              "sample": f"per step {nwin} windows x 4096 consecutive configs spread over the sweep"},
                e2e={"value": v, "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                vs_baseline=None, scaling=args.scaling)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def ours(args):
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    n_gpus = ws
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_2104_09075_b200 as P
    from workloads import sweeps as W

    sweep = bench_sweep(args, dist_env()[0])
    ctx = P.Context(dev.index)
    spec = ctx.prepare(sweep)
    N = ctx.sweep_size(spec)
    stream = torch.cuda.current_stream()

    lists = torch.empty((max(ws, 1), K_TOP, 2), dtype=torch.int64, device=dev)
    counts = torch.zeros(max(ws, 1), dtype=torch.int64, device=dev)
    my_rec = torch.zeros((K_TOP + 1, 2), dtype=torch.int64, device=dev)   # k hits + count record
    my_hits = my_rec[:K_TOP]
    my_cnt = my_rec[K_TOP, :1]
    out = torch.empty((K_TOP, 2), dtype=torch.int64, device=dev)
    out_cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    launches = [0]

    from paper_2104_09075_b200 import dist as PD

    def step():
        if ws > 1:
            _, _, st_ = PD.sharded_topk(ctx, spec, 0, N, K_TOP, out, out_cnt, my_rec, stream=stream)
            launches[0] += st_["launches"]
            return out, out_cnt
        ctx.topk_async(spec, 0, N, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
        launches[0] += ctx.stat(2)
        return my_hits, my_cnt

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    sampler = ClockSampler(dev.index if "CUDA_VISIBLE_DEVICES" not in os.environ else local)
    sampler.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches[0] = 0
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)              # L2 flush between timed steps (not timed)
        evs[i][0].record(stream)
        res, rc = step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    value = N * args.steps / (t_ms * 1e-3)
    gpu_launches = launches[0]
    best = res.cpu().numpy()
    n_feasible = int(rc.item())
    best_hits = [(int(i) % (1 << 64), float(k)) for i, k in zip(best[:, 0], best[:, 1].view("float64"))]
    gold = golden_check(args.config, sweep, N, best_hits, n_feasible) if args.scaling == "strong" or ws == 1 else None

    # ---- e2e: public C-ABI, host inputs (spec image re-uploaded) and host results
    e2e_ms = []
    h2d = d2h = 0
    if ws == 1:
        for i in range(args.warmup + args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            ctx.set_system(sweep.system)          # invalidates the resident image -> H2D each step
            hits, nf = ctx.topk(spec, K_TOP, 0, N, stream=stream)
            h2d, d2h = ctx.stat(0), ctx.stat(1)
            t1.record(stream)
            t1.synchronize()
            if i >= args.warmup:
                e2e_ms.append(t0.elapsed_time(t1))
        assert nf == n_feasible and hits[0][0] == int(best[0, 0]) % (1 << 64)
    else:
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            ctx.set_system(sweep.system)
            _, _, st_ = PD.sharded_topk(ctx, spec, 0, N, K_TOP, out, out_cnt, my_rec, stream=stream)
            h2d = st_["h2d"]
            host = out.cpu()
            _ = out_cnt.cpu()
            d2h = host.numel() * 8 + 8
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            if i >= args.warmup:
                e2e_ms.append(float(dt.item()) * 1e3)
    e2e_value = N * len(e2e_ms) / (sum(e2e_ms) * 1e-3)

    # ---- roofline of the dominant kernel (pipeline family: 78,600 of 79,051 configs per outer tuple)
    roof = None
    fp64_peak = ctx.fp64_peak(60.0)
    # dominant kernel: the largest sub-sweep of the workload (cfg2: the pipeline family)
    sizes = []
    for i, sb in enumerate(sweep.subs):
        sizes.append((sub_spec(P, spec, sweep, i), i))
    sizes = [(ctx.sweep_size(sp), i, sp) for sp, i in sizes]
    ctx.set_system(sweep.system)
    dom = max(sizes, key=lambda t: t[0])[1:] if sizes else None
    if dom is not None:
        di, dspec = dom
        fam_name = W.FAMILY_NAMES[sweep.subs[di].family]
        nd = ctx.sweep_size(dspec)
        for _ in range(3):
            ctx.topk_async(dspec, 0, nd, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
        kev = []
        for i in range(10 if nd < 1e10 else 3):
            flush.fill_(2)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            ctx.topk_async(dspec, 0, nd, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
            b_.record(stream)
            kev.append((a_, b_))
        torch.cuda.synchronize()
        kms = statistics.mean(a.elapsed_time(b) for a, b in kev)
        n_feas = int(my_cnt.item())
        # algorithmic FP64 work: the cost tree runs for feasible configurations only (the
        # others are rejected by integer / single-compare checks before any FP64 work)
        opc = fp64_per_config(sweep.subs[di])
        ops = n_feas * opc
        achieved = ops / (kms * 1e-3) / 1e12
        peak = fp64_peak / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(f"sweep_kernel_{fam_name}_bytes_per_launch")
            except Exception:
                traffic = None
        ncu_fp = None
        fp_path = os.path.join(ROOT, "profiles", "fp64_ncu.json")
        if os.path.exists(fp_path):
            try:
                ncu_fp = json.load(open(fp_path)).get(sweep.name, {}).get(fam_name)
                ncu_fp = float(ncu_fp) if ncu_fp is not None else None
            except Exception:
                ncu_fp = None
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "T fp64-pipe inst/s",
                "fp64_inst_per_config_ncu": ncu_fp,
                "frac": achieved / peak, "traffic": traffic,
                "kernel": f"sweep_kernel<{fam_name.upper()},reduce> (+merge)", "configs_per_launch": nd,
                "fp64_inst_per_config": opc, "feasible_configs": n_feas,
                "launch_ms": kms,
                "peak_source": "measured DFMA-chain microbenchmark (paradl_fp64_peak) in this run",
                "peak_nominal_T": 148 * 64 * 1.965e9 / 1e12,
                "frac_of_nominal": achieved / (148 * 64 * 1.965e9 / 1e12),
                "configs_per_s": nd / (kms * 1e-3)}
        ctx.set_system(sweep.system)

    # ---- dense mode (a9): HBM-write-bound secondary figure
    dense = None
    if not args.no_dense and ws == 1:
        # a9 dense / compact writes on a cfg2 window (lane-strided tiles, alpha/beta blocks of
        # 4096: the evaluation is cheap next to the 17 B/config written)
        dsw = W.config2()
        spec = ctx.prepare(dsw)
        Nd = ctx.sweep_size(spec)
        cnt = 1 << 28
        t = torch.empty(cnt, dtype=torch.float64, device=dev)
        m = torch.empty(cnt, dtype=torch.float64, device=dev)
        bits = torch.empty(cnt // 32, dtype=torch.int32, device=dev)
        rs = torch.empty(cnt, dtype=torch.uint8, device=dev)
        first = Nd // 3
        for _ in range(2):
            ctx.sweep_dense(spec, first, cnt, t.data_ptr(), m.data_ptr(), bits.data_ptr(), rs.data_ptr(), stream=stream)
        dv = []
        for _ in range(5):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            ctx.sweep_dense(spec, first, cnt, t.data_ptr(), m.data_ptr(), bits.data_ptr(), rs.data_ptr(), stream=stream)
            b_.record(stream)
            dv.append((a_, b_))
        torch.cuda.synchronize()
        dms = statistics.mean(a.elapsed_time(b) for a, b in dv)
        nbytes = cnt * (8 + 8 + 1) + cnt // 8
        # write-only reference measured here (a plain device fill): the copy peak in
        # MEASURED_PEAKS.json counts reads + writes, a write-only stream tops out lower
        wbuf = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
        wbuf.fill_(1)
        fv = []
        for _ in range(3):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            wbuf.fill_(2)
            b_.record(stream)
            fv.append((a_, b_))
        torch.cuda.synchronize()
        wpeak = (4 << 30) / (min(a.elapsed_time(b) for a, b in fv) * 1e-3) / 1e9
        del wbuf
        ach = nbytes / (dms * 1e-3) / 1e9
        # compact mode: feasible-only (idx, t_iter, mem) in index order, same window
        cidx = torch.empty(cnt, dtype=torch.int64, device=dev)
        cnf = torch.zeros(1, dtype=torch.int64, device=dev)
        for _ in range(2):
            ctx.sweep_compact(spec, first, cnt, cidx.data_ptr(), cnt, cnf.data_ptr(), t.data_ptr(), m.data_ptr(),
                              stream=stream)
        cv = []
        for _ in range(5):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            ctx.sweep_compact(spec, first, cnt, cidx.data_ptr(), cnt, cnf.data_ptr(), t.data_ptr(), m.data_ptr(),
                              stream=stream)
            b_.record(stream)
            cv.append((a_, b_))
        torch.cuda.synchronize()
        cms = statistics.mean(a.elapsed_time(b) for a, b in cv)
        cnf_v = int(cnf.item())
        cbytes = cnf_v * 24
        del cidx
        compact = {"configs": cnt, "feasible": cnf_v, "ms": cms, "configs_per_s": cnt / (cms * 1e-3),
                   "bytes_per_feasible_config": 24, "write_GBps": cbytes / (cms * 1e-3) / 1e9,
                   "passes": "count per tile + scan, then write (the evaluation runs twice)"}
        dense = {"workload": dsw.name, "window": [first, cnt], "compact": compact,
                 "configs": cnt, "ms": dms, "configs_per_s": cnt / (dms * 1e-3),
                 "write_GBps": ach, "bytes_per_config": 17.125, "bound": "hbm",
                 "write_only_peak_GBps_measured": wpeak, "frac_of_write_peak": ach / wpeak,
                 "copy_peak_GBps": 6538.3, "frac_of_copy_peak": ach / 6538.3}
        del t, m, bits, rs

    nxt = None
    if ws == 1 and not args.no_next:
        nxt = next_rows(ctx, P, W, stream, flush, my_hits, my_cnt, fp64_peak)
        ctx.set_system(sweep.system)

    per_cfg = None
    if ws == 1 and not args.no_configs:
        per_cfg = config_lines(ctx, P, W, stream, flush, my_hits, my_cnt, fp64_peak, args.config)
        ctx.set_system(sweep.system)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(sweep, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC if args.scaling == "strong" or ws == 1 else METRIC_WEAK,
            "value": value, "unit": "configs/s", "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(sweep, N, ws),
            "e2e": {"value": e2e_value, "unit": "configs/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(gpu_launches),
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "dense": dense,
            "next_rows": nxt,
            "result": {"argmin_idx": int(best[0, 0]) % (1 << 64), "n_feasible": n_feasible, "vs_oracle_golden": gold},
            "configs": per_cfg,
            "fp64_peak_inst_per_s": fp64_peak,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def dominant_roofline(ctx, P, W, sweep, spec, stream, flush, my_hits, my_cnt, fp64_peak, reps=3):
    """FP64 roofline of the largest sub-sweep of `sweep`, timed alone (L2 flushed)."""
    import torch
    sizes = [(ctx.sweep_size(sub_spec(P, spec, sweep, i)), i) for i in range(len(sweep.subs))]
    nd, di = max(sizes)
    dspec = sub_spec(P, spec, sweep, di)
    fam = W.FAMILY_NAMES[sweep.subs[di].family]
    ctx.topk_async(dspec, 0, nd, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
    ev = []
    for _ in range(reps):
        flush.fill_(5)
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        ctx.topk_async(dspec, 0, nd, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
        b_.record(stream)
        ev.append((a_, b_))
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    nf = int(my_cnt.item())
    opc = fp64_per_config(sweep.subs[di])
    ach = nf * opc / (ms * 1e-3) / 1e12
    ncu_fp = None
    try:
        v = json.load(open(os.path.join(ROOT, "profiles", "fp64_ncu.json"))).get(sweep.name, {}).get(fam)
        ncu_fp = float(v) if v is not None else None
    except Exception:
        pass
    return {"bound": "alu", "kernel": f"sweep_kernel<{fam.upper()},reduce>", "sub_sweep_configs": nd,
            "launch_ms": ms, "fp64_inst_per_config": opc, "fp64_inst_per_config_ncu": ncu_fp,
            "achieved": ach, "peak": fp64_peak / 1e12,
            "unit": "T fp64-pipe inst/s", "frac": ach / (fp64_peak / 1e12)}


def config_lines(ctx, P, W, stream, flush, my_hits, my_cnt, fp64_peak, headline):
    """The other BASELINE configs, each one whole-sweep top-64 + count per
    step timed like the headline (L2 flushed before each timed launch), with the FP64 roofline
    of its largest sub-sweep and the comparison with its oracle golden where one exists."""
    import torch
    out = {}
    for cfg in sorted(W.CONFIGS):
        if cfg == headline:
            continue
        sw = W.CONFIGS[cfg]()
        spec = ctx.prepare(sw)
        n = ctx.sweep_size(spec)
        reps = 3 if n > 5e10 else 10
        ctx.topk_async(spec, 0, n, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
        evs = []
        for _ in range(reps):
            flush.fill_(4)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            ctx.topk_async(spec, 0, n, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
            b_.record(stream)
            evs.append((a_, b_))
        torch.cuda.synchronize()
        ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
        nf = int(my_cnt.item())
        h = my_hits.cpu().numpy()
        hits = [(int(i) % (1 << 64), float(k)) for i, k in zip(h[:, 0], h[:, 1].view("float64"))]
        line = {"workload": sw.name, "configs": n, "ms": ms, "configs_per_s": n / (ms * 1e-3),
                "result": {"argmin_idx": hits[0][0], "n_feasible": nf,
                           "vs_oracle_golden": golden_check(cfg, sw, n, hits, nf)}}
        if n > 1000:
            line["roofline"] = dominant_roofline(ctx, P, W, sw, spec, stream, flush, my_hits, my_cnt, fp64_peak)
        out[f"cfg{cfg}"] = line
    return out


def gpipe_ops(s: int, S: int) -> int:
    """FP64 instructions of one GPipe schedule evaluation: boundary costs
    c_i = alpha + m_i beta (2 per boundary), busy times f_i + c_i and g_i + c_{i-1} (2 per
    boundary), one add per (segment, stage) in each wave and one max per (segment > 0,
    stage with an upstream neighbour) -- the other maxima of the event simulation are
    provably against a smaller operand --, then s adds and s-1 maxima for the WU ends and
    the key multiply."""
    return 4 * (s - 1) + 2 * s * S + 2 * (s - 1) * (S - 1) + s + (s - 1) + 1


def next_rows(ctx, P, W, stream, flush, my_hits, my_cnt, fp64_peak):
    """SURVEY §8(f) rows built this round, timed like the headline sweep (top-64 + count
    over the whole sweep, L2 flushed before each timed launch): the GPipe schedule family
    (f3) and the spatial prefix + Allgather family (f4)."""
    import torch
    out = {}
    for name, fn in W.NEXT.items():
        sw = fn()
        spec = ctx.prepare(sw)
        n = ctx.sweep_size(spec)
        for _ in range(3):
            ctx.topk_async(spec, 0, n, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
        evs = []
        for i in range(5):
            flush.fill_(3)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            ctx.topk_async(spec, 0, n, 0, 1, K_TOP, my_hits.data_ptr(), my_cnt.data_ptr(), stream=stream)
            b_.record(stream)
            evs.append((a_, b_))
        torch.cuda.synchronize()
        ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
        n_feas = int(my_cnt.item())
        best = int(my_hits[0, 0].item()) % (1 << 64)
        if name == "gpipe":
            # exact algorithmic count: S varies faster than the partition and only decides
            # SEGMENTS, so each (b, stage count) block's feasible count = feasible partitions x
            # feasible S x alpha/beta; the per-config work depends on (s, S)
            sb = sw.subs[0]
            G = sw.models[0].G
            nS, nAB = len(sb.S), len(sb.alpha) * len(sb.beta)
            blk = [math.comb(G - 1, s - 1) for s in range(sb.s_min, sb.s_max + 1)]
            per_b = sum(blk) * nS * nAB
            ops = 0.0
            for bi, b in enumerate(sb.b):
                Sok = [S for S in sb.S if S <= b]
                off = 0
                for j, s in enumerate(range(sb.s_min, sb.s_max + 1)):
                    first = bi * per_b + off * nS * nAB
                    cnt_ = blk[j] * nS * nAB
                    _, c = ctx.topk(spec, 1, first, cnt_)
                    if Sok:
                        n_pf = c / (len(Sok) * nAB)
                        ops += n_pf * nAB * sum(gpipe_ops(s, S) for S in Sok)
                    off += blk[j]
            opc = ops / max(1, n_feas)
            kern = "sweep_kernel<GPIPE,reduce>"
        elif name == "data_lw":
            # per configuration: 4 FP64 per weighted layer (s*beta, alpha+, c*, fold +), comp +
            # GE, key * I; exact per sub-sweep (models differ in weighted layers)
            ops = 0.0
            for si, sb in enumerate(sw.subs):
                lw = sum(1 for r in sw.models[sb.model].layers if r.w > 0)
                ss = sub_spec(P, spec, sw, si)
                _, c = ctx.topk(ss, 1, 0, ctx.sweep_size(ss))
                ops += c * (4.0 * lw + 2.0)
            ctx.prepare(sw)
            opc = ops / max(1, n_feas)
            kern = "sweep_kernel<DATA_LW,reduce>"
        elif name == "layerwise":
            opc = FP64_OPS_PER_CONFIG["layerwise"]
            ops = opc * n_feas
            kern = "sweep_kernel<LAYERWISE,reduce>"
        else:
            opc = FP64_OPS_PER_CONFIG["spatial_ag"]   # GE 3 + Allgather 3 + halo 3 + 1/M + key 1
            ops = opc * n_feas
            kern = "sweep_kernel<SPATIAL_AG,reduce>"
        ach = ops / (ms * 1e-3) / 1e12
        out[name] = {"workload": sw.name, "configs": n, "ms": ms, "configs_per_s": n / (ms * 1e-3),
                     "n_feasible": n_feas, "argmin_idx": best, "kernel": kern,
                     "roofline": {"bound": "alu", "achieved": ach, "peak": fp64_peak / 1e12,
                                  "unit": "T fp64-pipe inst/s", "frac": ach / (fp64_peak / 1e12),
                                  "fp64_inst_per_config": opc}}
    return out


def sub_spec(P, spec, sweep, i):
    """C spec of sub-sweep i alone (model ids as loaded for the whole sweep)."""
    mids = {sb.model: spec.c.sub[j].model_id for j, sb in enumerate(sweep.subs)}
    return P.Spec([sweep.subs[i]], mids)


def spec_model_id(ctx, spec, sub_index):
    return spec.c.sub[sub_index].model_id


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
