"""BASELINE config 4: neglect-threshold sweep on the c4 geometry (512 units).

usage:
  python tools/tau_sweep.py time [taus...]          -> one JSON line per tau (device-timed)
  python tools/tau_sweep.py one TAU                 -> one fourfold build (for an ncu pass)
  python tools/tau_sweep.py report time.jsonl ncu_TAU.csv...  -> merged table (JSON)

Per tau: tau_ovlp = 1e-3 tau (configs.config4); fourfold driver.  Surviving-quartet
fraction = eri_shell_quartets / (canonical shell pairs)^2, canonical pair = (i <= j) of
the ns shells (the fourfold driver's quartet universe, before overlap pruning).  The
culling-stage HBM GB/s (k_expand + k_screen2) and ERI-stage FP64 utilisation (k_eri,
dadd + dmul + 2 dfma per thread instruction) come from an ncu metric pass of `one`
(gpu__time_duration, dram__bytes_read/write, sm__sass_thread_inst_executed_op_d*).
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

TAUS = (1e-4, 1e-6, 1e-8, 1e-10)


def _build(tau, reps):
    import torch
    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import configs, exchange
    cfg = configs.config4(tau_2e=tau)
    part = hx.build_partition(cfg.system, cfg.leaf_size)
    part.device(0)
    pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
    ns = cfg.n_shells
    Pd = torch.as_tensor(cfg.P, device="cuda")
    Kd = torch.empty_like(Pd)
    out = []
    for _ in range(reps):
        Pt = hx.build_matrix_tree(Pd, part)
        _, c, _ = exchange.run_exchange(pairs, pairs, Pt, tau, "schwarz", True, K_out=Kd)
        torch.cuda.synchronize()
        out.append((c, exchange.last_timings()))
        del Pt
    return cfg, ns, out


def cmd_time(taus):
    for tau in taus:
        cfg, ns, runs = _build(tau, 3)
        c, t = runs[-1]
        best = min(r[1][4] for r in runs[1:])
        npair = ns * (ns + 1) // 2
        q = int(c.eri_shell_quartets)
        print(json.dumps({
            "tau_2e": tau, "tau_ovlp": cfg.tau_ovlp, "shells": ns,
            "surviving_quartets": q, "prim_quartets": int(c.prim_quartets),
            "surviving_fraction": q / float(npair * npair),
            "k_build_ms": best, "quartets_per_s": q / (best * 1e-3),
            "stage_ms": {"traversal": t[0], "leaf_screen": t[1], "eri_stage": t[2], "epilogue": t[3]},
            "tasks_visited": int(c.tasks_visited), "ties_task": int(c.ties_task), "ties_leaf": int(c.ties_leaf),
        }), flush=True)


def cmd_one(tau):
    _build(tau, 1)


_UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_groups(path):
    """Sum ncu metrics over the culling kernels and the ERI kernels of one capture."""
    hdr, g = None, {"cull": {}, "eri": {}}
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        grp = "eri" if "k_eri" in name else ("cull" if ("k_expand" in name or "k_screen2" in name) else None)
        if grp is None:
            continue
        m = d["Metric Name"]
        v = float(d["Metric Value"].replace(",", "")) * _UNIT.get(d["Metric Unit"], 1.0)
        g[grp][m] = g[grp].get(m, 0.0) + v
    return g


def cmd_report(time_path, ncu_paths, peak_fp64, peak_hbm):
    rows = [json.loads(l) for l in open(time_path) if l.strip().startswith("{")]
    for row in rows:
        p = [x for x in ncu_paths if x.endswith("_%g.csv" % row["tau_2e"])]
        if not p:
            continue
        g = ncu_groups(p[0])
        cu, er = g["cull"], g["eri"]
        tb = cu.get("dram__bytes_read.sum", 0) + cu.get("dram__bytes_write.sum", 0)
        tt = cu.get("gpu__time_duration.sum", 0)
        f = (er.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
             + er.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
             + 2 * er.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0))
        te = er.get("gpu__time_duration.sum", 0)
        row["ncu"] = {
            "culling_dram_bytes": tb, "culling_kernel_ms": 1e3 * tt,
            "culling_hbm_gbs": tb / tt / 1e9 if tt else None,
            "culling_hbm_frac": tb / tt / 1e9 / peak_hbm if tt else None,
            "eri_fp64_flops_executed": f, "eri_kernel_ms": 1e3 * te,
            "eri_fp64_tflops": f / te / 1e12 if te else None,
            "eri_fp64_frac": f / te / 1e12 / peak_fp64 if te else None,
        }
    print(json.dumps({"config": "c4 (512 units, c3 recipe), fourfold", "peak_fp64_tflops": peak_fp64,
                      "peak_hbm_gbs": peak_hbm, "rows": rows}, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "time":
        cmd_time([float(x) for x in sys.argv[2:]] or TAUS)
    elif cmd == "one":
        cmd_one(float(sys.argv[2]))
    elif cmd == "report":
        peak_f = float(os.environ.get("PEAK_FP64", "36.7"))
        peak_h = float(os.environ.get("PEAK_HBM", "6542.1"))
        cmd_report(sys.argv[2], sys.argv[3:], peak_f, peak_h)
    else:
        raise SystemExit(__doc__)
