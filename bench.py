"""Benchmark: surviving ERI quartets/s and K-build ms of the hierarchical exchange build.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` (torchrun for
N>1) prints ONE JSON line on rank 0.  A step is one exchange build of the
workload: density quadtree from a device-resident P + traversal + leaf
screening + ERIs + contraction into K (+ NCCL all-reduce of K and the fourfold
epilogue for N>1).  The shell-pair tree is geometry-only (built once per
SCF) and is reported separately as `pair_tree_ms`.

`--impl reference` times the reference's own CPU implementation (hexfock,
installed unmodified into baseline/_ref, which travels to the GPU box) on a
bounded s-only sub-cluster of the same recipe (the reference has no p shells),
the faster of threads=1 and threads=cpu_count, rank 0 only; the p-capable
oracle port on the full basis is reported beside it.  Without baseline/_ref
the port stands in (kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ERI_FLOPS = os.path.join(ROOT, "paper_1401_6961_b200", "csrc", "eri_flops.json")
# executed FP64 flops per primitive quartet per class, measured once with ncu
# (tools/fp64_rate.py); the SURVEY 8(d) graded rate for the p classes
ERI_FLOPS_EXEC = os.path.join(ROOT, "profiles", "r01_eri_fp64_executed.json")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "surviving ERI quartets/s (FP64 exchange K-build)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--units", type=int, default=None, help="override cluster size (c3-c5 recipe)")
    ap.add_argument("--mode", default="fourfold", choices=["naive", "fourfold", "eightfold"],
                    help="eightfold: the 4-fold build folded bra<->ket (same K, ~half the quartets; "
                         "no reference counterpart, the CPU baseline runs the 4-fold port)")
    ap.add_argument("--tau", type=float, default=None)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample-units", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-eightfold", action="store_true",
                    help="fourfold runs: skip the companion eightfold K-build timing")
    return ap.parse_args()


def make_config(args, device_density=False):
    from paper_1401_6961_b200 import configs
    kw = {}
    if args.units is not None:
        if args.config in ("c1", "c2"):
            raise SystemExit("--units applies to the cube recipes c3-c5")
        kw["n_units"] = args.units
    if args.config in ("c3", "c4", "c5") and device_density:
        kw["host_density"] = False      # generated on the GPU below
    cfg = configs.make(args.config, **kw)
    if args.tau is not None:
        cfg.tau_2e = args.tau
        cfg.tau_ovlp = 1e-3 * args.tau
    return cfg


def workload_desc(args, cfg):
    d = {"workload": f"{args.config}" + (f"-{args.units}units" if args.units else ""),
         "mode": args.mode, "shells": cfg.n_shells, "functions": cfg.n_functions,
         "tau_2e": cfg.tau_2e, "tau_ovlp": cfg.tau_ovlp, "leaf_size": cfg.leaf_size,
         "bound": "schwarz", "basis": "s3/s1/p2 heavy + s3 light" if args.config != "c1" else "s3"}
    return d


# --------------------------------------------------------------- CPU baselines

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _import_reference():
    """The unmodified reference package (hexfock 0.1.0) installed into baseline/_ref
    (pip --target from a copy of /root/reference/pkg), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "hexfock")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import hexfock  # noqa: F401
        from hexfock import basis, exchange_naive, exchange_symmetry, quadtree
    except Exception:
        return None
    return basis, quadtree, exchange_naive, exchange_symmetry


def ref_sample(args):
    """The reference's own CPU path needs s shells, so it runs on the
    s-only sub-basis of the workload's recipe: the same geometry recipe, s shells
    only, the matching rows / columns of the same density.
    c1 is all-s and runs in full; c3-c5 use a bounded sub-cluster."""
    from paper_1401_6961_b200 import configs
    if args.config == "c1":
        cfg = configs.config1()
        desc = "full c1 (32 s shells)"
    elif args.config == "c2":
        n = args.cpu_sample_units or 48
        cfg = configs.config2(n_centers=n)
        desc = f"c2 recipe, {n}-center chain"
    else:
        n = args.cpu_sample_units or 16
        cfg = configs.cube_cluster(n, {"c3": 3, "c4": 4, "c5": 5}[args.config], args.config)
        desc = f"{args.config} cube recipe, {n} units"
    if args.tau is not None:
        cfg.tau_2e = args.tau
        cfg.tau_ovlp = 1e-3 * args.tau
    return cfg, desc


def run_reference_cpu(args, steps):
    """Time the reference's build_exchange_symmetric / build_exchange_naive
    (exchange_symmetry.py:364, exchange_naive.py:200) on the host cores.  Trees
    are built once, outside the timed builds (cli.py times them together; we
    report them apart).  Both threads=1 and threads=os.cpu_count() are run (the
    reference farms depth-1 subtrees over a thread pool, GIL-bound); the faster
    is the reported value and the timed steps use it.  None if baseline/_ref is
    not installed."""
    import numpy as np
    mods = _import_reference()
    if mods is None:
        return None
    hb, hq, hn, hs = mods
    cfg, desc = ref_sample(args)
    sh = cfg.system.shells
    fn = np.concatenate([[0], np.cumsum([s.n_functions for s in sh])])
    keep = [k for k, s in enumerate(sh) if int(getattr(s, "l", 0)) == 0]
    fidx = np.asarray([fn[k] for k in keep])
    shells = [hb.GaussianShell(center=sh[k].center, primitives=list(sh[k].primitives)) for k in keep]
    system = hb.BasisSystem(shells=hb._assign_offsets(shells), atoms=[])
    P = np.ascontiguousarray(np.asarray(cfg.P)[np.ix_(fidx, fidx)])
    t0 = time.perf_counter()
    part = hq.build_partition(system, cfg.leaf_size)
    pairs = hq.build_pair_tree(system, part, tau_ovlp=cfg.tau_ovlp)
    P_tree = hq.build_matrix_tree(P, part)
    tree_ms = 1e3 * (time.perf_counter() - t0)
    naive = args.mode == "naive"

    def build(threads):
        t = time.perf_counter()
        if naive:
            _, c = hn.build_exchange_naive(pairs, pairs, P_tree, tau_2e=cfg.tau_2e, threads=threads)
        else:
            _, c = hs.build_exchange_symmetric(pairs, P_tree, tau_2e=cfg.tau_2e, threads=threads)
        return time.perf_counter() - t, c.eri_shell_quartets

    nall = os.cpu_count() or 1
    t1, q = build(1)
    tall, _ = build(nall)
    best = 1 if t1 <= tall else nall
    times = [build(best)[0] for _ in range(steps)] if steps else [min(t1, tall)]
    tot = sum(times)
    return {"value": q * len(times) / tot, "unit": "quartets/s", "cores": best, "kind": "reference",
            "sample": (desc + f", s-only sub-basis: {len(shells)} s shells of {cfg.n_shells}, "
                       f"{len(shells)} functions; {q} surviving quartets per build, "
                       f"{1e3 * tot / len(times):.0f} ms per build"),
            "impl": ("hexfock 0.1.0 (unmodified, baseline/_ref) "
                     + ("build_exchange_naive" if naive else "build_exchange_symmetric")),
            "threads_1": {"quartets_per_s": q / t1, "ms_per_build": 1e3 * t1},
            "threads_all": {"cores": nall, "quartets_per_s": q / tall, "ms_per_build": 1e3 * tall},
            "tree_build_ms": tree_ms,
            "note": "the faster of threads=1 / threads=cpu_count is reported; the reference cannot "
                    "evaluate p shells, so its rate is on the s-only sub-basis"}


def port_sample(args):
    """Bounded sample of the full (p-shell) workload for the oracle port."""
    from paper_1401_6961_b200 import configs
    if args.config == "c1":
        return configs.config1(), "full c1 (32 s shells)"
    if args.config == "c2":
        n = 24
        return configs.config2(n_centers=n), f"c2 recipe, {n}-center chain"
    n = 6
    cfg = configs.cube_cluster(n, {"c3": 3, "c4": 4, "c5": 5}[args.config], args.config)
    return cfg, f"{args.config} cube recipe, {n} units ({cfg.n_shells} shells, {cfg.n_functions} functions)"


def run_port_cpu(args):
    """One build of the oracle port (oracle/hexfock_oracle.py, p-capable) with the
    full basis, single-threaded (its thread pool is GIL-bound)."""
    from oracle import hexfock_oracle as ho
    cfg, desc = port_sample(args)
    if args.tau is not None:
        cfg.tau_2e, cfg.tau_ovlp = args.tau, 1e-3 * args.tau
    st = ho.Setup(cfg.system, cfg.P, tau_ovlp=cfg.tau_ovlp, leaf_size=cfg.leaf_size)
    f = st.naive if args.mode == "naive" else st.symmetric
    t0 = time.perf_counter()
    _, c = f(cfg.tau_2e, threads=1)
    dt = time.perf_counter() - t0
    return {"value": c.eri_shell_quartets / dt, "unit": "quartets/s", "cores": 1, "kind": "port",
            "sample": desc + f"; {c.eri_shell_quartets} surviving quartets per build, {1e3 * dt:.0f} ms per build"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warmup = args.steps, min(args.warmup, 1)
    cb = run_reference_cpu(args, steps)
    port = None
    if cb is None:   # baseline/_ref absent: the oracle port stands in
        cb = run_port_cpu(args)
        note = "oracle port of the reference algorithm (baseline/_ref not installed)"
    else:
        port = run_port_cpu(args)
        note = ("the reference's own CPU implementation (" + cb["impl"] + ") on a bounded s-only "
                "sample of the workload; warm-up = one threads=1 and one threads=cpu_count build")
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "quartets/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "mode": "naive" if args.mode == "naive" else "fourfold",
                       "note": note},
            "cpu_baseline": cb,
            "port_full_basis": port,
            "e2e": {"value": cb["value"], "unit": "quartets/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU

class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region.

    NVML from a background thread every 500 ms (light: two queries per sample);
    falls back to `nvidia-smi -lms 500` when pynvml is unavailable.  A 200 ms
    nvidia-smi poll measurably slowed the timed steps (~2 %).
    """
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index = index
        self.samples = []      # (sm_mhz, max_mhz, reasons bitmask)
        self.proc = None
        self.nvml = None
        self.stop_evt = threading.Event()

    def start(self):
        if os.environ.get("HXF_BENCH_NO_CLOCKS"):  # diagnostic: no sampling thread
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            self.nvml = pynvml

            def loop():
                while not self.stop_evt.is_set():
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, get_r(h)))
                    except Exception:
                        pass
                    self.stop_evt.wait(0.5)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "500"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7 and parts[0].replace(".", "").isdigit():
                mask = 0
                for k, (_, bit) in enumerate(self.REASONS):
                    if parts[3 + k].lower() in ("active", "1"):
                        mask |= bit
                mx = float(parts[1]) if parts[1].replace(".", "").isdigit() else 0.0
                self.samples.append((float(parts[0]), mx, mask))

    def stop(self):
        if self.nvml is not None:
            self.stop_evt.set()
            self.thread.join(timeout=5)
        elif self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(s[0]) for s in self.samples]
        mx = [float(s[1]) for s in self.samples]
        reasons = sorted({name for s in self.samples for name, bit in self.REASONS if int(s[2]) & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def eri_flops_executed(c):
    try:
        tab = json.load(open(ERI_FLOPS_EXEC))["per_prim"]
    except (OSError, ValueError, KeyError):
        return None
    if any(c.class_prim_quartets[k] and tab[k] is None for k in range(16)):
        return None
    return sum(c.class_prim_quartets[k] * (tab[k] or 0.0) for k in range(16))


def eri_flops(c):
    tab = json.load(open(ERI_FLOPS))
    return sum(c.class_prim_quartets[k] * tab["per_prim"][k] + c.class_quartets[k] * tab["per_quartet"][k]
               for k in range(16))


def ncu_traffic(workload, mode):
    """Per-build DRAM bytes of the path's kernels from the newest committed ncu
    metric pass of this workload (profiles/*_ncu_<workload>_dram.json, written by
    tools/ncu_dram.py), or None."""
    import glob
    here = os.path.dirname(os.path.abspath(__file__))
    for path in sorted(glob.glob(os.path.join(here, "profiles", f"*_ncu_{workload}_dram.json")), reverse=True):
        with open(path) as fh:
            d = json.load(fh)
        if d.get("mode") == mode:
            d["file"] = os.path.relpath(path, here)
            return d
    return None


def hbm_peak():
    """Measured copy bandwidth (GB/s) from the driver-written MEASURED_PEAKS.json, else None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return None


def native_arm(args):
    import ctypes
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import _native, distributed, exchange

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    t0 = time.perf_counter()
    cfg = make_config(args, device_density=True)
    if cfg.P is None:
        from paper_1401_6961_b200 import configs
        P_gen = configs.decay_density_device(cfg.system, cfg.density_seed, dev)
        torch.cuda.synchronize()
    else:
        P_gen = None
    gen_s = time.perf_counter() - t0
    sym = "eightfold" if args.mode == "eightfold" else args.mode == "fourfold"
    part = hx.build_partition(cfg.system, leaf_size=cfg.leaf_size)
    part.device(local)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=cfg.tau_ovlp)
    torch.cuda.synchronize()
    pair_ms = 1e3 * (time.perf_counter() - t0)
    n = cfg.n_functions
    if P_gen is None:
        P_host = torch.from_numpy(cfg.P).pin_memory()
        P_dev = P_host.to(dev)
    else:
        P_dev = P_gen
        P_host = torch.empty((n, n), dtype=torch.float64).pin_memory()
        P_host.copy_(P_dev)
    K_dev = torch.empty((n, n), dtype=torch.float64, device=dev)
    K_host = torch.empty((n, n), dtype=torch.float64).pin_memory()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    l2_flush = cfg.n_functions ** 2 * 8 < 256 * 1024 * 1024

    peak = ctypes.c_double(0.0)
    _native.check(_native.lib().hxf_fp64_peak(ctypes.byref(peak), _native.current_stream()))

    shards = None
    plan_ms = None
    if world > 1:
        P_tree0 = hx.build_matrix_tree(P_dev, part)
        # once per geometry + density (an SCF reuses it across iterations): hashed task
        # groups, costs from counters-only builds (each rank measures 1/world of
        # them), longest-first onto ranks
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        shards = distributed.plan(pairs, pairs, P_tree0, cfg.tau_2e, "schwarz", sym, world,
                                  strategy="balanced", K_scratch=K_dev)
        torch.cuda.synchronize()
        plan_ms = 1e3 * (time.perf_counter() - t0)
        del P_tree0

    def step(P_src):
        P_tree = hx.build_matrix_tree(P_src, part)
        if world > 1:
            c, _ = distributed.exchange_sharded(pairs, pairs, P_tree, cfg.tau_2e, "schwarz", sym,
                                                K_dev, shards=shards)
            return c
        _, c, _ = exchange.run_exchange(pairs, pairs, P_tree, cfg.tau_2e, "schwarz", sym, True,
                                        None, K_out=K_dev)
        return distributed.counters_from_vector(distributed.counters_vector(c), bool(sym))

    for _ in range(args.warmup):
        step(P_dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    lc0 = ctypes.c_int64(0)
    _native.lib().hxf_launch_count(ctypes.byref(lc0))
    clocks = ClockSampler(local)
    clocks.start()
    times, stage, quartets, flops, last = [], [], 0, 0.0, None
    stream = torch.cuda.current_stream()
    for _ in range(args.steps):
        if l2_flush:
            flush.fill_(1.0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c = step(P_dev)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        stage.append(exchange.last_timings())
        last = c
    clk = clocks.stop()
    lc1 = ctypes.c_int64(0)
    _native.lib().hxf_launch_count(ctypes.byref(lc1))

    # max over ranks of the timed region
    tt = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total_ms = float(tt.item())
    quartets = last.eri_shell_quartets
    value = quartets * args.steps / (total_ms * 1e-3)

    # roofline: ERI + contraction kernels on the FP64 pipe (this rank)
    _, cl, _ = (None, None, None)
    # re-run once with the hxf counters struct for per-class work (untimed)
    P_tree = hx.build_matrix_tree(P_dev, part)
    shard = None
    if world > 1:
        lv, rng = shards
        shard = (lv,) + tuple(rng[rank])
    _, craw, _ = exchange.run_exchange(pairs, pairs, P_tree, cfg.tau_2e, "schwarz", sym, True, None,
                                       K_out=K_dev, shard=shard, symmetrize=not (world > 1), screen_bytes=True)
    tm = exchange.last_timings()
    flops = eri_flops(craw)
    flops_exec = eri_flops_executed(craw)
    eri_ms = statistics.median([s[5] for s in stage]) if stage else tm[5]
    achieved = flops / (eri_ms * 1e-3) / 1e12 if eri_ms > 0 else 0.0
    achieved_exec = flops_exec / (eri_ms * 1e-3) / 1e12 if (eri_ms > 0 and flops_exec) else None

    # e2e through the drop-in API a reference caller uses (N = 1): a pageable numpy
    # P into build_matrix_tree (H2D inside), build_exchange_symmetric /
    # build_exchange_naive / build_exchange_eightfold, numpy K out (D2H inside),
    # timed with the host clock between device synchronisations.  N > 1: the
    # sharded step from pinned host P (the drop-in has no multi-GPU entry point).
    e2e_times = []
    if world == 1:
        P_np = np.array(P_host.numpy(), copy=True)      # pageable host copy, made once
        build = {"naive": lambda Pt: hx.build_exchange_naive(pairs, pairs, Pt, tau_2e=cfg.tau_2e),
                 "fourfold": lambda Pt: hx.build_exchange_symmetric(pairs, Pt, tau_2e=cfg.tau_2e),
                 "eightfold": lambda Pt: hx.build_exchange_eightfold(pairs, Pt, tau_2e=cfg.tau_2e)}[args.mode]
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Pt = hx.build_matrix_tree(P_np, part)
            K_np, c_e2e = build(Pt)
            torch.cuda.synchronize()
            e2e_times.append(1e3 * (time.perf_counter() - t0))
            del Pt
            assert c_e2e.eri_shell_quartets == quartets
        del P_np
        K_np = None
        e2e_api = "drop-in: build_matrix_tree(numpy P) + build_exchange_" + \
            {"naive": "naive", "fourfold": "symmetric", "eightfold": "eightfold"}[args.mode] + \
            " -> numpy K (pageable host buffers)"
    else:
        P_in = torch.empty_like(P_dev)
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            P_in.copy_(P_host, non_blocking=True)
            step(P_in)
            K_host.copy_(K_dev, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_times.append(e0.elapsed_time(e1))
        e2e_api = "exchange_sharded from pinned host P, K to pinned host"
    et = torch.tensor([sum(e2e_times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = quartets * args.e2e_steps / (float(et.item()) * 1e-3) if args.e2e_steps else None

    # companion eightfold build (same K, bra<->ket folded): K-build time, folded
    # quartet count, and max |K8 - K4| against the fourfold K of the timed steps
    eight = None
    if args.mode == "fourfold" and world == 1 and not args.no_eightfold:
        K4 = K_dev.clone()
        K8 = torch.empty_like(K_dev)
        e8 = []
        c8 = None
        for it in range(1 + args.steps):
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            Pt8 = hx.build_matrix_tree(P_dev, part)
            _, c8, _ = exchange.run_exchange(pairs, pairs, Pt8, cfg.tau_2e, "schwarz", "eightfold", True,
                                             None, K_out=K8)
            a1.record(stream)
            torch.cuda.synchronize()
            del Pt8
            if it:  # the first is a warm-up
                e8.append(a0.elapsed_time(a1))
        ms8 = statistics.median(e8)
        eight = {"k_build_ms": ms8, "surviving_quartets_per_step": int(c8.eri_shell_quartets),
                 "prim_quartets_per_step": int(c8.prim_quartets),
                 "fourfold_quartets_per_s": quartets / (ms8 * 1e-3),
                 "max_abs_diff_vs_fourfold_K": float((K8 - K4).abs().max().item()),
                 "note": "same K as the fourfold build (bra<->ket folded, K = A + A^T); "
                         "fourfold_quartets_per_s = the fourfold surviving-quartet count / this K-build time"}
        del K4, K8

    cpu = port = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_reference_cpu(args, 0)
        port = run_port_cpu(args)
        if cpu is None:
            cpu, port = port, None

    if rank == 0:
        stage_med = [statistics.median([s[k] for s in stage]) for k in range(7)] if stage else tm
        nt = ncu_traffic(args.config, args.mode) if world == 1 else None
        hbm = hbm_peak()
        # traversal: SURVEY 8(d) algorithmic bytes per visited task (naive 48 B, symmetric 104 B)
        bpt = 48 if args.mode == "naive" else 104
        trav_gbs = bpt * last.tasks_visited / (stage_med[0] * 1e-3) / 1e9 if stage_med[0] > 0 else None
        roof_trav = {"bound": "hbm", "achieved": trav_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": trav_gbs / hbm if (trav_gbs and hbm) else None,
                     "traffic": nt["k_expand"]["dram_bytes_per_build"] if nt else None,
                     "kernel": "k_expand (count + write passes), all levels",
                     "bytes_basis": f"algorithmic: {bpt} B per visited task (SURVEY 8(d)) x tasks_visited",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy test)",
                     "traffic_source": nt["file"] if nt else None}
        # leaf screen: SURVEY 8(d) algorithmic bytes (Q of both pair lists + the |P| block of
        # every live slot per leaf task, counted by the kernel) + the 8-byte record and 2-byte
        # key written per surviving quartet, over the screen's device time
        screen_bytes = int(craw.screen_bytes) + 10 * int(craw.eri_shell_quartets)
        screen_gbs = screen_bytes / (stage_med[1] * 1e-3) / 1e9 if stage_med[1] > 0 else None
        scr_traffic = (nt.get("k_screen2") or nt.get("k_screen") or {}).get("dram_bytes_per_build") if nt else None
        roof_screen = {"bound": "hbm", "achieved": screen_gbs, "peak": hbm, "unit": "GB/s",
                       "frac": screen_gbs / hbm if (screen_gbs and hbm) else None,
                       "traffic": scr_traffic,
                       "kernel": "k_screen2 (hierarchical leaf screen), all chunks",
                       "bytes_basis": "algorithmic: 8 (m_bra + m_ket) B of Q + 8 n_row n_col B of |P| per live slot "
                                      "per leaf task (SURVEY 8(d), counted on the device: screen_bytes) "
                                      "+ 10 B per surviving quartet (record + sort key)",
                       "bytes_per_step_rank0": screen_bytes,
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy test)",
                       "traffic_source": nt["file"] if nt else None,
                       "note": "the node vectors and |P| blocks the screen gathers are L2-resident and the "
                               "kernel is instruction-issue bound (ncu: issue active 66 %, DRAM ~130 GB/s), "
                               "so the HBM fraction is low by construction; see DESIGN.md"}
        roof_trav["dram_gbs_ncu"] = (roof_trav["traffic"] / (stage_med[0] * 1e-3) / 1e9
                                     if (roof_trav["traffic"] and stage_med[0] > 0) else None)
        roof_trav["note"] = ("achieved = algorithmic bytes / stage time; the node arrays are L2-resident, so the "
                             "DRAM rate ncu measures (dram_gbs_ncu) is ~20x lower and the kernel is issue-bound: "
                             "not an HBM utilisation")
        line = {
            "metric": METRIC, "value": value, "unit": "quartets/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64 geometry + decay density, SURVEY Appendix B)",
            "config": dict(workload_desc(args, cfg), parallelism=f"product-tree shards x{world}",
                           l2=("256 MB flush between steps" if l2_flush else
                               "inputs larger than L2 (P alone exceeds 126 MB)")),
            "k_build_ms": total_ms / args.steps,
            "surviving_quartets_per_step": quartets,
            "prim_quartets_per_step": last.prim_quartets,
            "stage_ms": {"traversal": stage_med[0], "leaf_screen": stage_med[1],
                         "eri_stage": stage_med[2], "epilogue": stage_med[3],
                         "exchange_total": stage_med[4], "eri_kernels": stage_med[5],
                         "far_classify_and_sort": stage_med[6]},
            "pair_tree_ms": pair_ms, "input_gen_s": gen_s,
            "counters": last.to_dict() | {"ties_task": last.ties_task, "ties_leaf": last.ties_leaf},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value,
                         "unit": "TFLOP/s", "frac": achieved / peak.value if peak.value else None,
                         "traffic": nt["k_eri"]["dram_bytes_per_build"] if nt else None,
                         "traffic_source": (nt["file"] + ": dram__bytes_read.sum + dram__bytes_write.sum "
                                            "over the k_eri launches of one build") if nt else None,
                         "kernel": "k_eri<la,lb,lc,ld> (ERI + contraction), all classes",
                         "flops_per_step_rank0": flops,
                         "peak_source": "hxf_fp64_peak DFMA microbenchmark on this GPU "
                                        "(MEASURED_PEAKS.json has no FP64 entry)",
                         "flops_basis": "algorithmic: 30 per (ss|ss) primitive quartet (SURVEY 8(d)), "
                                        "generated OS/HGP operation counts for the p classes, "
                                        "executed (non-neglected) primitive quartets"},
            "roofline_executed": {"bound": "fp64", "achieved": achieved_exec, "peak": peak.value,
                                  "unit": "TFLOP/s",
                                  "frac": (achieved_exec / peak.value) if (achieved_exec and peak.value) else None,
                                  "flops_basis": "executed FP64 (dadd + dmul + 2 dfma) per primitive quartet "
                                                 "per class from ncu, profiles/r01_eri_fp64_executed.json"},
            "roofline_traversal": roof_trav,
            "roofline_screen": roof_screen,
            "plan_ms": plan_ms,
            "e2e": {"value": e2e_value, "unit": "quartets/s",
                    "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": n * n * 8,
                    "ms_per_step": float(et.item()) / max(args.e2e_steps, 1), "api": e2e_api},
            "cpu_baseline": cpu,
            "cpu_port_full_basis": port,
            "eightfold": eight,
            "gpu_launches": int(lc1.value - lc0.value),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        native_arm(args)


if __name__ == "__main__":
    main()
