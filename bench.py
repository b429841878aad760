#!/usr/bin/env python
"""CF-operator apply benchmark (BASELINE.json metric: applies/s and points/s).

One step = one combined-field operator apply out = 1/2 phi + D[phi] - i gamma S[phi]
(CombinedOperator::apply, solver.cpp:149-157). Default workload: cfg3, the 64-wavelength
sphere (N = 6,291,456), the BASELINE config quoted at 1/2/4/8 GPUs that fits one B200
(SURVEY.md Appendix A maps BASELINE's 6 x 1024^2 layout to the reference-constructible
24,576 x 16^2 patches with the same N). --config cfg1/cfg2 select the smaller spheres.

  value : points/s with phi resident in HBM (CUDA-graph replays timed with CUDA events on
          the engine stream), whole job (sum over ranks, max time over ranks)
  e2e   : the same through the public API with host buffers — pinned phi copied in and the
          result read back every step (CombinedOperator.apply)
  roofline / rooflines : per-phase device time (CUDA events) against the algorithmic work
  cpu_baseline : the reference (oracle/_ref, built from the untouched /root/reference
          sources) on the host's cores: cfg1/cfg2 one full CombinedOperator::apply; cfg3 a
          bounded sample (ifgf_apply + the near-field loop, run at cfg2)
  parity : cfg1/cfg2 the reference's full apply with its OWN beta tables; cfg3 the committed
          reference fixture tests/golden/cfg3_large.npz (64 random projections of S and D
          over all N, 65,536 sampled targets, the RP term of 16,384 targets from the
          reference's own beta tables) — see tests/golden/large_check.py

--impl reference runs the reference CPU implementation alone (rank 0), same metric/config;
at cfg3 one step = the reference's ifgf_apply + near-field loop (its beta tables would need
101 GB and hours), one timed step after an untimed setup.
--gpus N without a torchrun environment re-launches itself under torch.distributed.run.
Multi-GPU (torchrun): one operator per GPU over a cost-balanced Morton partition of the
sources/targets, far-field partials reduced and outputs broadcast with NCCL inside the
engine; the same N-point apply at every N, scaling "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

# torch.distributed.run exports OMP_NUM_THREADS=1 to its workers when several run on a node.
# The host side of the setup (cone plan, proximity, mesh) is OpenMP code: every local rank
# gets its share of the cores instead, and the reference arm (rank 0 alone) all of them.
# Set before anything loads an OpenMP runtime.
_LWS = int(os.environ.get("LOCAL_WORLD_SIZE", "1") or 1)
if _LWS > 1:
    _ref_arm = any(a == "reference" or a == "--impl=reference" for a in sys.argv[1:])
    os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or 1) // (1 if _ref_arm else _LWS)))

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (splits, nodes per patch side, k, gamma, description); SPHEROIDS adds the axes
    "cfg1": (2, 16, 4 * np.pi, 4 * np.pi, "sphere r=1, 4 wavelengths, 96 patches x 16^2, k=4pi, gamma=k"),
    "cfg2": (4, 16, 16 * np.pi, -1.0, "sphere r=1, 16 wavelengths, 1536 patches x 16^2, k=16pi"),
    "cfg3": (6, 16, 64 * np.pi, -1.0, "sphere r=1, 64 wavelengths, 24576 patches x 16^2, k=64pi"),
    "cfg4": (6, 16, 2 * np.pi, -1.0, "spheroid (40,4,4) lambda=1, 24576 patches x 16^2, k=2pi"),
    # BASELINE configs[4] (a GMRES solve on 8 B200s; 406 GB of beta tables: >= 3 GPUs)
    "cfg5": (7, 16, 128 * np.pi, -1.0, "sphere r=1, 128 wavelengths, 98304 patches x 16^2, k=128pi"),
}
SPHEROIDS = {"cfg4": (40.0, 4.0, 4.0)}  # cube-sphere coefficients scaled


def make_mesh(cfg_name, module):
    """the config's surface from the product (paper_2112_06316_b200) or the oracle (oracle.ref)"""
    splits, nu = CONFIGS[cfg_name][:2]
    cls = module.SurfaceMesh if hasattr(module, "SurfaceMesh") else module.RefMesh
    if cfg_name in SPHEROIDS:
        return cls.spheroid(splits, nu, nu, *SPHEROIDS[cfg_name])
    return cls.sphere(1.0, splits, nu, nu)


def peaks():
    p = {"hbm_gbs": 6551.4, "fp64_tflops": 36.9,
         "source_fp64": "highest FP64 rate measured on this pool's B200: 8 DMMA chains per warp, tools/fp64_mix.cu "
                        "(profiles/r02ag_fp64_mix.json: DMMA 36.9, DFMA 36.4 TF/s, one shared pipe; "
                        "tools/fp64_peak.cu had 34.2 with 8 DFMA chains)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p["hbm_gbs"] = float(m.get("hbm_gbs", p["hbm_gbs"]))
        p["source_hbm"] = "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        p["hbm_gbs"] = 6650.0
        p["source_hbm"] = "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent)"
    return p


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], None, set()
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 7:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx = float(f[1])
                except ValueError:
                    continue
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                for nm, v in zip(names, f[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except Exception:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def barrier_max(value, ws):
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reference_apply_time(cfg_name, phi, beta_cache=None, applies=1, warmup=0):
    """Times the reference's own CombinedOperator::apply; returns (seconds list, out, setup_s)."""
    from oracle import ref as R

    splits, nu, k, gamma, _ = CONFIGS[cfg_name]
    rm = make_mesh(cfg_name, R)
    t0 = time.perf_counter()
    ro = R.RefOperator(rm, k, gamma=gamma, beta_cache=beta_cache or "")
    setup = time.perf_counter() - t0
    for _ in range(warmup):
        ro.apply(phi)
    times = []
    out = None
    for _ in range(applies):
        t0 = time.perf_counter()
        out = ro.apply(phi)
        times.append(time.perf_counter() - t0)
    return times, out, setup, R.lib().ref_op_beta_cache_hit(ro.h) == 1


LARGE = {"cfg3", "cfg4", "cfg5"}
BETA_GB = {"cfg3": 101, "cfg4": 178, "cfg5": 406}  # no reference beta tables: ifgf_apply + near loop


def reference_ifgf_near_time(cfg_name, phi, steps=1):
    """The reference's ifgf_apply + near-field loop (layer_potentials without its RP term) on
    a plan built without beta tables; returns (seconds list, S, D, setup dict)."""
    from oracle import ref as R

    splits, nu, k, gamma, _ = CONFIGS[cfg_name]
    rm = make_mesh(cfg_name, R)
    t0 = time.perf_counter()
    rp = R.RefPlan(rm, k, gamma=gamma)
    setup = dict(rp.setup_seconds, total=time.perf_counter() - t0)
    times, S, D = [], None, None
    for _ in range(steps):
        S, D, sec = rp.ifgf_near(phi)
        times.append(sec["ifgf_apply"] + sec["near"])
    return times, S, D, setup


def run_reference(args, ws, rank):
    cfg_name = args.config
    splits, nu, k, gamma, desc = CONFIGS[cfg_name]
    if rank != 0:
        return
    n = 6 * 4 ** splits * nu * nu
    from oracle import ref as R

    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libifgf_ref.so not built"}))
        return
    phi = R.random_density(n, 1)
    cores = os.cpu_count()
    if cfg_name == "cfg5":
        print(json.dumps({"impl": "reference", "unavailable": "cfg5 (N = 25.2 M): the reference's setup alone takes "
                          "hours on the host cores and its GMRES basis ~20 GB; no CPU baseline (SURVEY.md 8(d))"}))
        return
    if cfg_name in LARGE:
        steps, warm = 1, 0
        times, _, _, setup = reference_ifgf_near_time(cfg_name, phi, steps)
        total = sum(times)
        value = n * steps / total
        sample = (f"1 step = the reference's ifgf_apply (ifgf.cpp:577-608) + the level-D near-field loop "
                  f"(solver.cpp:100-144) at {cfg_name} (N={n}), i.e. CombinedOperator::layer_potentials minus "
                  f"its RP term: the reference's beta tables would need {BETA_GB.get(cfg_name, '100+')} GB and hours of "
                  f"CPU (BASELINE.md §3); "
                  f"setup (octree, plan_cones, classify_targets) {setup['total']:.0f} s untimed; OpenMP {cores} "
                  f"threads; 1 step, no warm-up, to bound the run")
        line = {
            "impl": "reference", "metric": "cf_operator_points_per_s", "value": value, "unit": "points/s",
            "applies_per_s": steps / total, "n_gpus": args.gpus, "steps": steps, "warmup": warm,
            "steps_requested": args.steps, "ms_per_step": 1e3 * total / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": f"{cfg_name}: {desc}", "N": n, "k": k, "parallelism": "cpu-openmp"},
            "setup_s": setup,
            "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return
    steps = max(1, min(args.steps, args.ref_steps))
    warm = min(args.warmup, 1)
    times, _, setup, _ = reference_apply_time(cfg_name, phi, applies=steps, warmup=warm)
    total = sum(times)
    value = n * steps / total
    line = {
        "impl": "reference", "metric": "cf_operator_points_per_s", "value": value, "unit": "points/s",
        "applies_per_s": steps / total, "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "steps_requested": args.steps, "ms_per_step": 1e3 * total / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"{cfg_name}: {desc}", "N": n, "k": k, "parallelism": "cpu-openmp"},
        "setup_s": setup,
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "reference",
                         "sample": f"{steps} full CombinedOperator::apply at {cfg_name} after {warm} warm-up"
                                   f" (reference built from /root/reference sources, OpenMP {cores} threads);"
                                   f" steps capped at {args.ref_steps} to bound the run"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def roofline_for(phases, work, pk):
    """per-phase achieved rates; fp64 roof for leaf/near, HBM for cousin/parent/rp (north_star)"""
    m = {
        "leaf": ("leaf_flops", "leaf_bytes", "fp64"),
        "cousin": ("cousin_flops", "cousin_bytes", "hbm"),
        "parent": ("parent_flops", "parent_bytes", "hbm"),
        "near": ("near_flops", "near_bytes", "fp64"),
        "rp": ("rp_flops", "rp_bytes", "hbm"),
    }
    out = {}
    for ph, (fk, bk, bound) in m.items():
        ms = phases.get(ph, 0.0)
        if ms <= 0:
            continue
        tf = work[fk] / (ms * 1e-3) / 1e12
        gbs = work[bk] / (ms * 1e-3) / 1e9
        out[ph] = {"ms": ms, "fp64_tflops": tf, "fp64_frac": tf / pk["fp64_tflops"], "hbm_gbs": gbs,
                   "hbm_frac": gbs / pk["hbm_gbs"], "stated_bound": bound,
                   "flops": work[fk], "bytes": work[bk]}
    return out


KERNEL_FAMILY = {"leaf": ("leaf_ray_kernel",), "cousin": ("cousin_tc_kernel",), "parent": ("parent_tc_kernel", "parent_cb_kernel"),
                 "near": ("near_list_kernel", "near_pair_kernel"), "rp": ("rp_accum_kernel",)}


def ncu_traffic(cfg_name, phase):
    """dram__bytes_read.sum + dram__bytes_write.sum per apply of the phase's kernel from the newest
    committed ncu launch list for this config (profiles/r*_ncu_launches_<cfg>.json, written by
    tools/ncu_launches.py); None when there is none."""
    import glob

    def tag_key(f):  # r02g < r02z < r02aa < r02ad: round, then tag length, then tag
        import re

        m = re.match(r"r(\d+)([a-z]*)_", os.path.basename(f))
        return (int(m.group(1)), len(m.group(2)), m.group(2)) if m else (0, 0, "")

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_launches_{cfg_name}.json")), key=tag_key)
    if not files:
        return None, None
    try:
        ks = json.load(open(files[-1]))["kernels"]
        got = [ks[f]["dram_bytes_per_apply"] for f in KERNEL_FAMILY[phase] if f in ks]
        return (sum(got) if got else None), os.path.relpath(files[-1], ROOT)
    except Exception:
        return None, None


def check_parity(cfg_name, op, phi, out_gpu):
    """cfg1/cfg2: the reference's full CombinedOperator::apply with its own beta tables,
    compared over all N. cfg3: the committed reference fixture (large_check.py)."""
    if cfg_name in LARGE:
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        import large_check as LC

        path = os.path.join(ROOT, "tests", "golden", f"{cfg_name}_large.npz")
        if not os.path.exists(path):
            return {"parity": {"error": f"no reference fixture for {cfg_name} (tests/golden/make_large.py)"}}
        fix = np.load(path)
        if not np.array_equal(phi[:8], fix["phi_head"]):
            raise RuntimeError("density differs from the fixture's")
        S, D = op.layer_potentials(phi)
        rS, rD = op.rp_singular_apply(phi)
        res = LC.compare(fix, S - rS, D - rD)
        idx = fix["rp_idx"]
        rp = LC.compare_rp(fix, rS[idx], rD[idx])
        # out at the RP-sampled targets from the reference's S, D and RP terms
        g = float(fix["gamma"])
        s_ref = fix["S_sample"][np.searchsorted(fix["sample_idx"], idx)] + fix["rpS"]
        d_ref = fix["D_sample"][np.searchsorted(fix["sample_idx"], idx)] + fix["rpD"]
        out_ref = 0.5 * phi[idx] + d_ref - 1j * g * s_ref
        out_rel = float(np.linalg.norm(out_gpu[idx] - out_ref) / np.linalg.norm(out_ref))
        head = max(res["S"]["rel_l2_est_full"], res["D"]["rel_l2_est_full"], out_rel)
        return {"rel_l2_vs_reference": head, "parity": {
            "method": "reference fixture tests/golden/cfg3_large.npz (tests/golden/make_large.py from oracle/_ref): "
                      "S, D without RP over ALL N via 64 random projections (estimated rel-L2), exact on 65,536 "
                      "sampled targets; RP from the reference's own beta_precompute + rp_singular_apply on 16,384 "
                      "targets; out on those targets",
            "S_D_noRP": res, "rp_sample": rp, "out_rel_l2_rp_sample": out_rel,
            "fixture_ref_seconds": json.loads(str(fix["ref_seconds"]))}}
    from oracle import ref as R

    if not R.available():
        return {"parity": {"error": "oracle/_ref not built"}}
    times, out_ref, setup = _ref_full(cfg_name, phi)
    rel = float(np.linalg.norm(out_gpu - out_ref) / np.linalg.norm(out_ref))
    return {"rel_l2_vs_reference": rel,
            "parity": {"method": f"reference CombinedOperator::apply at {cfg_name} over all N with its own "
                                 f"beta_precompute (setup {setup:.1f} s)",
                       "max_abs": float(np.max(np.abs(out_gpu - out_ref)))}}


_REF_FULL = {}


def _ref_full(cfg_name, phi):
    """one reference CombinedOperator (own beta tables) per config: (apply times, out, setup s)"""
    if cfg_name not in _REF_FULL:
        times, out, setup, _ = reference_apply_time(cfg_name, phi, applies=1)
        _REF_FULL[cfg_name] = (times, out, setup)
    return _REF_FULL[cfg_name]


def cpu_baseline(cfg_name, n):
    """The reference on the host's cores (reported, not the target)."""
    from oracle import ref as R

    if not R.available():
        return {"error": "oracle/_ref not built"}
    cores = os.cpu_count()
    if cfg_name in LARGE:  # bounded sample: ifgf_apply + near loop at cfg2 (~20 s on 16 cores)
        sub = "cfg2"
        m = 6 * 4 ** CONFIGS[sub][0] * CONFIGS[sub][1] ** 2
        times, _, _, setup = reference_ifgf_near_time(sub, R.random_density(m, 1), 1)
        return {"value": m / times[0], "unit": "points/s", "cores": cores, "kind": "reference",
                "seconds": times[0],
                "sample": f"bounded sample: the reference's ifgf_apply + near-field loop (BASELINE.md §3; no RP: "
                          f"its {cfg_name} beta tables would need 100+ GB) on the cfg2 sphere "
                          f"(N={m}, 1/16 of {cfg_name}'s points; the reference's per-point cost grows ~log N, so this "
                          f"overstates its {cfg_name} rate); OpenMP {cores} threads; --impl reference times "
                          f"{cfg_name} itself"}
    times, _, setup = _ref_full(cfg_name, R.random_density(n, 1))
    return {"value": n / times[0], "unit": "points/s", "cores": cores, "kind": "reference", "seconds": times[0],
            "sample": f"one full CombinedOperator::apply at {cfg_name} (N={n}), reference built from /root/reference "
                      f"sources, OpenMP {cores} threads, its own beta tables (setup {setup:.1f} s)"}


def spawn_ranks(args):
    """--gpus N outside torchrun: re-launch this command under torch.distributed.run"""
    import socket

    import torch

    if torch.cuda.device_count() < args.gpus:
        print(json.dumps({"metric": "cf_operator_points_per_s", "n_gpus": args.gpus,
                          "error": f"--gpus {args.gpus} but {torch.cuda.device_count()} GPU(s) visible"}))
        sys.exit(1)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def run_b200(args, ws, rank, local):
    import torch

    import paper_2112_06316_b200 as P

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    splits, nu, k, gamma, desc = CONFIGS[args.config]
    t0 = time.perf_counter()
    mesh = make_mesh(args.config, P)
    cfg = P.SolveConfig(k=k, gamma=gamma, device=local)
    if ws > 1:  # one operator per GPU, Morton-partitioned, NCCL exchange inside the engine
        from paper_2112_06316_b200.distributed import DistributedCombinedOperator

        op = DistributedCombinedOperator(mesh, cfg)
    else:
        op = P.CombinedOperator(mesh, cfg)
    setup_s = time.perf_counter() - t0
    n = mesh.size()
    phi = P.random_density(n, 1)

    # --- device-resident throughput
    op.upload_density(phi)
    op.time_applies(max(args.warmup, 3), flush_l2=False)  # warm-up (eager run + graph capture)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as cs:
        t_wall = time.perf_counter()
        each = op.time_applies_each(args.steps, flush_l2=False)
        t_wall = time.perf_counter() - t_wall
    ms_per = float(np.mean(each))
    torch.cuda.synchronize()
    clocks = cs.summary()
    ms_per = barrier_max(ms_per, ws)
    value = n / (ms_per * 1e-3)  # one N-point apply per step, whole job

    # --- end to end through the public API with pinned host buffers
    pin_in = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
    pin_out = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
    phi_h = pin_in.numpy().view(np.complex128)
    phi_h[:] = phi
    out_h = pin_out.numpy().view(np.complex128)
    for _ in range(max(args.warmup, 3)):
        op.apply_into(phi_h, out_h)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t_e2e = time.perf_counter()
    for _ in range(args.steps):
        op.apply_into(phi_h, out_h)
    t_e2e = time.perf_counter() - t_e2e
    t_e2e = barrier_max(t_e2e, ws)
    e2e_value = n * args.steps / t_e2e
    out_gpu = out_h.copy()

    # --- phases, work, roofline
    phases = op.time_phases()
    work = op.work()
    pk = peaks()
    roofs = roofline_for(phases, work, pk)
    dom = max(roofs, key=lambda p: roofs[p]["ms"])
    r = roofs[dom]
    traffic, traffic_src = ncu_traffic(args.config, dom)
    # north_star: HBM GB/s is the stated roofline of the propagation / SpMV kernels and FP64 of
    # the leaf / near-field kernels; the FP64 pipe is what binds the propagation kernels
    # (SURVEY.md 8(d)), so both fractions are reported
    binding = {"bound": "fp64", "achieved": r["fp64_tflops"], "peak": pk["fp64_tflops"], "unit": "TFLOP/s",
               "frac": r["fp64_frac"], "peak_source": pk["source_fp64"]}
    if r["stated_bound"] == "fp64":
        roof = dict(binding, kernel=dom, traffic=traffic)
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": r["hbm_gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": r["hbm_frac"], "traffic": traffic, "peak_source": pk["source_hbm"], "binding": binding}
    roof["algorithmic_bytes"] = r["bytes"]
    roof["algorithmic_flops"] = r["flops"]
    roof["per"] = "one apply (all launches of the kernel: one per level)"
    roof["traffic_source"] = traffic_src

    line = {
        "metric": "cf_operator_points_per_s", "value": value, "unit": "points/s",
        "applies_per_s": 1.0 / (ms_per * 1e-3), "n_gpus": ws, "steps": args.steps, "warmup": max(args.warmup, 3),
        "ms_per_step": ms_per, "ms_best": float(np.min(each)), "ms_median": float(np.median(each)),
        "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None,
        "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"{args.config}: {desc}", "N": n, "k": k, "gamma": op.gamma,
                   "density": "U(-1,1)+iU(-1,1), mt19937_64 seed 1",
                   "parallelism": f"morton-partitioned x{ws} (NCCL reduce/broadcast)" if ws > 1 else "single",
                   "l2": "no flush: each apply streams the plan + beta tables (>> 126 MB L2)"},
        "setup_s": setup_s, "setup_breakdown_s": op.setup_times(), "wall_s_timed": t_wall, "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 16 * n, "ms_per_step": 1e3 * t_e2e / args.steps},
        "gpu_launches": args.steps * op.kernels_per_apply(), "kernels_per_apply": op.kernels_per_apply(),
        "phases_ms": phases, "work": work, "roofline": roof, "rooflines": roofs,
    }

    # --- parity + CPU baseline at the bench config (rank 0, N=1; outside the timed regions)
    if rank == 0 and ws == 1 and not args.no_check:
        try:
            line.update(check_parity(args.config, op, phi, out_gpu))
        except Exception as e:  # report, never hide
            line["parity"] = {"error": repr(e)}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config, n)
        except Exception as e:
            line["cpu_baseline"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=list(CONFIGS), default="cfg3")
    ap.add_argument("--ref-steps", type=int, default=3, help="cap on timed reference applies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the parity check against the reference")
    args = ap.parse_args()
    ws, rank, local = dist_setup()
    if args.impl == "b200" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_b200(args, ws, rank, local)


if __name__ == "__main__":
    main()
