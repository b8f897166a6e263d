#!/usr/bin/env python
"""Benchmark of one design-update pass (filter -> eta -> projection -> SIMP +
lower-triangle stiffness values -> sensitivity from a supplied U ->
back-filter -> OC bisection) on B200, BASELINE.json's metric:
Melem/s per pass, FP64, with the HBM-roofline fraction.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

N > 1 is launched by torchrun (one rank per GPU, x-slab decomposition of the
same grid: strong scaling). Rank 0 prints ONE JSON line.

Timing: W untimed passes, then K passes bracketed by barrier + synchronize,
timed with CUDA events on the context's stream (device time, max over ranks).
Inputs are resident in HBM and larger than L2 for C4/C5 (C5 writes 34 GB of
stiffness values per pass); for C1-C3 the L2 is flushed between passes.
e2e repeats the measurement through the C-ABI with pinned HOST buffers (H2D of
x and U, D2H of xNew and the scalars inside the timed region).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Melem/s per design-update pass (assemble+filter+sens+OC), FP64; % HBM roofline"
UNIT = "Melem/s"


def algorithmic_bytes_per_elem(cfg) -> float:
    """What one benchmarked pass must move at least: read x
    and U once, write sK and xNew [+ the state byte]. The timed pass requests
    no xPhys / dc / dV output, and the fused kernels never materialise them
    (the reference's Eigen temporaries), so they are not counted."""
    b = 8 + 8.0 * cfg.n / cfg.m + 8 * cfg.P + 8
    if cfg.passives:
        b += 1
    return b


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(cid: int):
    """ncu dram bytes per sK-store launch, committed under profiles/ (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"C{cid}", {}).get("sk_store_dram_bytes")
    except Exception:
        return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi in a separate process, sampling every 200 ms during the timed
    region (B200_PROFILING.md clocks line); no in-process NVML calls, which
    would contend with the CUDA driver on the timed thread."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        import shutil
        import subprocess
        import tempfile
        if shutil.which("nvidia-smi"):
            self.tmp = tempfile.TemporaryFile(mode="w+")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.tmp,
                stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.tmp.seek(0)
            self.lines = [ln.strip() for ln in self.tmp.read().splitlines() if ln.strip()]

    def summary(self):
        rows = []
        for ln in self.lines:
            f = [v.strip() for v in ln.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- CPU samples
def load_configs_standalone():
    """paper_2005_05436_b200/configs.py loaded as a plain module, with the
    oracle's copy of the Appendix B generator: the CPU reference arm never
    imports the product package, so no product library is mapped."""
    import importlib.util
    from oracle import oracle as O
    if not os.path.exists(O.PORT_LIB):
        O.build()
    spec = importlib.util.spec_from_file_location(
        "topo_configs_standalone", os.path.join(ROOT, "paper_2005_05436_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # (dataclasses resolve annotations through it)
    spec.loader.exec_module(mod)
    gen = O.Oracle("port")
    mod.set_generator(lambda seed, stream, kind, a, b, count, offset:
                      gen.generate(seed, stream, kind, a, b, count, offset))
    return mod


# Sample grids of the CPU legs: the config's physics, filter and OC parameters
# on a grid whose x extent is at least 2 reach + 1 (no mirror fold wraps a whole
# axis) and whose pass takes seconds on one core. The reference's per-element
# cost does not depend on the grid size at fixed taps: the filter is T taps per
# element per evaluation, and the number of OC volume evaluations is fixed by
# the regime (16 on C1-C3, 243 on C4/C5).
CPU_SAMPLES = {1: (300, 100, 0), 2: (150, 50, 0), 3: (70, 400, 0), 4: (12, 48, 48),
               5: (8, 32, 32)}


def cpu_sample_config(cfg):
    nx, ny, nz = CPU_SAMPLES.get(cfg.cid, (cfg.nelx, cfg.nely, cfg.nelz))
    return cfg.scaled(nx, ny, nz, name=f"{cfg.name} sample {nx}x{ny}x{nz}")


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"model": model, "nproc": os.cpu_count() or 1, "usable": usable}


def run_cpu(cfg, steps: int, warmup: int, threads: int, single: bool = True):
    """Times the reference CPU path (oracle/_ref = the reference's own headers
    compiled verbatim, else the C restatement): (ii) `threads` concurrent
    single-threaded sample passes, the reference having no threading on this
    path; (i) one pass alone on one core."""
    from oracle import oracle as O
    cmod = load_configs_standalone()
    kind = "reference" if os.path.exists(O.REF_LIB) else "port"
    orc = O.Oracle(kind)
    if kind == "port":
        orc.set_threads(1)
    scfg = cpu_sample_config(cfg)
    x, u, state = cmod.make_inputs(scfg)
    grid = scfg.grid
    mk = ((lambda: orc.problem(grid, scfg.rmin, 0, scfg.nu, state)) if kind == "reference"
          else (lambda: orc.filter(grid, scfg.rmin)))
    handles = [mk() for _ in range(threads)]

    def one(h):
        kw = dict(beta=scfg.beta, move=scfg.move, volfrac=scfg.volfrac)
        kw["problem" if kind == "reference" else "filt"] = h
        orc.design_pass(grid, scfg.rmin, x, u, state, **kw)

    def step(hs):
        ts = [threading.Thread(target=one, args=(h,)) for h in hs]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0

    for _ in range(warmup):
        step(handles)
    times = [step(handles) for _ in range(steps)]
    wall = sum(times) / len(times)
    value = threads * scfg.m / wall / 1e6
    res = {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
           "sec_per_step": wall, "host": host_cpu()}
    desc = (f"{scfg.nelx}x{scfg.nely}x{scfg.nelz} grid ({scfg.m} elements) with the "
            f"{cfg.name} filter / projection / OC parameters, literal ft=3 OC volume callback "
            f"(one filter per evaluation)")
    res["sample"] = (f"(ii) {threads} concurrent single-threaded passes of a {desc}, "
                     f"{steps} timed step(s)")
    if single:
        t1 = step(handles[:1])
        res["single_thread"] = {"value": scfg.m / t1 / 1e6, "unit": UNIT, "cores": 1,
                                "sec_per_pass": t1, "sample": f"(i) one pass of the same {desc}"}
    return res


# ------------------------------------------------------------------- ours
def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch
    import paper_2005_05436_b200 as P
    from paper_2005_05436_b200 import _lib as L
    from paper_2005_05436_b200.configs import make_inputs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    x, u, state = make_inputs(cfg)

    if world == 1:
        ctx = P.Context(*cfg.grid, rmin=cfg.rmin, nu=cfg.nu, device=local_rank, state=state)
    else:  # x-slab of this rank; halos and sums over NCCL (NVLink)
        from paper_2005_05436_b200.dist import make_rank_context, slab_views
        _, _, x, u, st = slab_views(cfg, x, u, state, rank, world)
        ctx = make_rank_context(cfg, st, rank, world, device=local_rank)
    m_local = ctx.m
    xd = torch.from_numpy(x).to(dev)
    ud = torch.from_numpy(u).to(dev)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)
    kw = dict(beta=cfg.beta, eta0=cfg.eta0, move=cfg.move, volfrac=cfg.volfrac, outputs=False)
    flush = None
    if cfg.m * algorithmic_bytes_per_elem(cfg) < 3 * 126e6:
        flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    stage_acc = {k: 0.0 for k in L.STAGES}
    launches = 0
    # warm-up = the timed step exactly (flush kernel loaded; the previous
    # result held while the next is allocated, so the caching allocator owns
    # both output blocks before timing starts)
    r = None
    for _ in range(args.warmup):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
        r = ctx.design_pass(xd, ud, **kw)
    barrier()
    torch.cuda.synchronize()
    # the timed call goes straight through the C-ABI (topo_design_pass as its
    # two halves, with the parameters ctx.design_pass(**kw) builds): _begin
    # enqueues the pass, the end event is recorded behind it on the stream,
    # _end waits and returns the scalars. The events bracket exactly the
    # device work of the pass (recorded after the synchronous call they would
    # also time the host's wake-up and the Python return, ~10% of a C4 pass)
    import ctypes as C
    import math
    pp = L.PassParams(P.SimpParams().c(), cfg.beta, cfg.eta0, cfg.move, cfg.volfrac, math.nan,
                      L.VOL_FILTERED, 1)
    xnew = torch.empty(m_local, dtype=torch.float64, device=dev)
    po = L.PassOut(None, None, None, None, None, xnew.data_ptr(), None)
    lib, h, xp, up = ctx.lib, ctx.h, xd.data_ptr(), ud.data_ptr()
    ppr, por = C.byref(pp), C.byref(po)
    for _ in range(max(1, args.warmup)):
        if lib.topo_design_pass(h, xp, up, ppr, por) != 0:
            raise RuntimeError("topo_design_pass failed")
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        t_total = 0.0
        for _ in range(args.steps):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(1.0)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            st = lib.topo_design_pass_begin(h, xp, up, ppr, por)  # enqueue only
            if world == 1:
                ev1.record(stream)
            st = st or lib.topo_design_pass_end(h, por)           # wait + scalars
            if world > 1:  # (multi-rank: _end may enqueue further OC batches)
                ev1.record(stream)
            ev1.synchronize()
            if st != 0:
                raise RuntimeError("topo_design_pass failed")
            t_total += ev0.elapsed_time(ev1)
            launches += ctx.launches
        torch.cuda.synchronize()
        barrier()
    # per-stage breakdown (CUDA events on each kernel's stream), measured in
    # extra passes after the timed region so the events do not perturb it
    ctx.set_timing(True)
    for _ in range(args.steps):
        ctx.design_pass(xd, ud, **kw)
        for k, v in ctx.stage_times().items():
            stage_acc[k] += v
    ctx.set_timing(False)
    ms = t_total / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64)  # gloo: host tensor
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stages = {k: v / args.steps for k, v in stage_acc.items()}

    # e2e through the C-ABI with pinned host buffers
    xh = torch.from_numpy(x).pin_memory()
    uh = torch.from_numpy(u).pin_memory()
    xnh = torch.empty(m_local, dtype=torch.float64).pin_memory()
    pp = L.PassParams(L.Simp(cfg.e0, cfg.emin, cfg.penal), cfg.beta, cfg.eta0, cfg.move,
                      cfg.volfrac, math.nan, L.VOL_FILTERED, 1)
    po = L.PassOut(None, None, None, None, None, xnh.data_ptr(), None)
    lib = ctx.lib
    for _ in range(max(1, args.warmup)):
        ctx._check(lib.topo_design_pass(ctx.h, xh.data_ptr(), uh.data_ptr(), C.byref(pp),
                                        C.byref(po)))
    barrier()
    torch.cuda.synchronize()
    e2e_ms = 0.0
    for _ in range(args.steps):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        ctx._check(lib.topo_design_pass_begin(ctx.h, xh.data_ptr(), uh.data_ptr(), C.byref(pp),
                                              C.byref(po)))
        if world == 1:
            ev1.record(stream)
        ctx._check(lib.topo_design_pass_end(ctx.h, C.byref(po)))
        if world > 1:
            ev1.record(stream)
        ev1.synchronize()
        e2e_ms += ev0.elapsed_time(ev1)
    e2e_ms /= args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = 8 * (x.size + u.size) * world
    d2h = (8 * m_local + 8 * 5) * world
    fp64 = None
    if rank == 0:  # FP64 DFMA peak of this GPU (the C2/C3 roof)
        t = C.c_double()
        if ctx.lib.topo_fp64_peak(local_rank, C.byref(t)) == 0:
            fp64 = t.value
    return dict(ms=ms, e2e_ms=e2e_ms, stages=stages, launches=launches, clocks=clk.summary(),
                h2d=h2d, d2h=d2h, r=r, m_local=m_local, flushed=flush is not None,
                ntaps=ctx.ntaps, fp64_peak=fp64)


def cpu_line(cb):
    out = {"value": cb["value"], "unit": UNIT, "cores": cb["cores"], "kind": cb["kind"],
           "sample": cb["sample"], "cpu_model": cb["host"]["model"],
           "nproc": cb["host"]["nproc"]}
    if "single_thread" in cb:
        out["single_thread"] = cb["single_thread"]
    return out


def launch_ranks(n: int) -> int:
    """`bench.py --gpus N` started without torchrun: start N ranks under
    torch.distributed.run (one per GPU, 127.0.0.1 rendezvous) and wait."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if args.impl == "ours":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                print(json.dumps({"error": f"--gpus {args.gpus} but {have} GPU(s) visible"}),
                      flush=True)
                sys.exit(2)
            sys.exit(launch_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE {world} != --gpus {args.gpus}"}), flush=True)
        sys.exit(2)
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        cfg = load_configs_standalone().CONFIGS[args.config]  # no product library
    else:
        from paper_2005_05436_b200.configs import CONFIGS
        cfg = CONFIGS[args.config]
    threads = args.cpu_threads or host_cpu()["usable"]
    workload = {"workload": cfg.name, "grid": list(cfg.grid), "m": cfg.m, "n_dofs": cfg.n,
                "rmin": cfg.rmin, "taps": None, "beta": cfg.beta, "move": cfg.move,
                "volfrac": cfg.volfrac, "filter_bc": "neumann (mirror)", "ft": 3,
                "parallelism": f"x-slab x{world}"}

    if args.impl == "reference":
        if rank != 0:
            return
        cb = run_cpu(cfg, args.steps, args.warmup, threads)
        workload["cpu_sample_grid"] = list(CPU_SAMPLES.get(cfg.cid, cfg.grid))
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": cb["sec_per_step"] * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload,
                "cpu_baseline": cpu_line(cb),
                "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group(backend="gloo")
    res = run_ours(args, cfg, rank, world, local_rank)
    if rank != 0:
        return
    peak, peak_kind = load_peaks()
    m = cfg.m
    value = m / (res["ms"] * 1e-3) / 1e6
    e2e_value = m / (res["e2e_ms"] * 1e-3) / 1e6
    # dominant kernel: K3b sK store (reads xTilde, writes m*P values)
    sk_ms = res["stages"]["sk_store"]
    sk_bytes = res["m_local"] * (8 * cfg.P + 8)
    sk_gbs = sk_bytes / (sk_ms * 1e-3) / 1e9 if sk_ms > 0 else None
    traffic = load_traffic(cfg.cid)
    b_elem = algorithmic_bytes_per_elem(cfg)
    pass_gbs = m * b_elem / (res["ms"] * 1e-3) / 1e9 / world  # per GPU
    # FP64 work per element: 3 convolutions x 2 T flops + the
    # sensitivity (2D 144, 3D 1200 as the dense form counts it)
    flop_elem = 6 * res["ntaps"] + (1200 if cfg.nelz else 144)
    fp64_tf = m * flop_elem / (res["ms"] * 1e-3) / 1e12 / max(1, world)
    workload["taps"] = res["ntaps"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded x~U(0.01,1), U~N(0,1); SURVEY.md Appendix B)",
        "config": dict(workload, l2=("flushed between passes (256 MiB write)" if res["flushed"]
                                     else "inputs/outputs larger than L2 (no flush)")),
        "roofline": {"bound": "hbm",
                     "kernel": ("k_sk_store_tma" if cfg.nelz and m * cfg.P * 8 >= 256e6
                                else "k_sk_store") + " (K3b, fea.hpp:135-146 + :162-169)",
                     "achieved": sk_gbs, "peak": peak, "unit": "GB/s",
                     "frac": (sk_gbs / peak) if sk_gbs else None, "traffic": traffic,
                     "bytes_per_launch": sk_bytes, "ms_per_launch": sk_ms,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"
                     if peak_kind == "measured" else "fallback 6650 GB/s (B200_PROFILING.md)"},
        "pass_roofline": {"bound": "hbm", "algorithmic_bytes_per_elem": b_elem,
                          "achieved": pass_gbs, "peak": peak, "unit": "GB/s",
                          "frac": pass_gbs / peak,
                          "ceiling_melem_s": peak * 1e9 / b_elem / 1e6 * world},
        "fp64_roofline": {"flop_per_elem": flop_elem, "achieved": fp64_tf,
                          "peak": res["fp64_peak"], "unit": "TFLOP/s",
                          "frac": fp64_tf / res["fp64_peak"] if res["fp64_peak"] else None,
                          "peak_source": "measured DFMA loop (topo_fp64_peak)"},
        "stages_ms": res["stages"],
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": res["h2d"],
                "d2h_bytes_per_step": res["d2h"], "ms_per_step": res["e2e_ms"]},
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "result": {"eta": res["r"].eta, "eta_iters": res["r"].eta_iters, "lambda": res["r"].lam,
                   "bisections": res["r"].bisections, "evaluations": res["r"].evaluations,
                   "c": res["r"].c},
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_line(run_cpu(cfg, 1, 0, threads))
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
