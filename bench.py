"""Benchmark of the JGS2 runtime iteration on B200 (driver contract).

A *step* is one JGS2 outer iteration (Jacobi sweep in corotated_cubature
mode incl. rotation refresh, exact reduced collect, sampled corrections,
local line search and the sweep-level backtracking guard), i.e. one
``LocalSolver.outer_solve`` iteration (reference local_solver.py:697-716).
``value`` = sweeps/s over all ranks with the state resident in HBM, in a
continuing simulation (frames end at tol_dx); ``sweeps`` carries the
backtracking statistics of the timed window (halvings histogram, floored
sweeps, accepted gamma/cap) and ``timestep`` whole frames to tol_dx.
``e2e`` = sweeps/s through the public API with host buffers: one
``LocalSolver.timestep`` (jgs2_timestep_host) per frame. The CPU oracle port
of the reference (numpy/SciPy, oracle/) is timed two ways:
``cpu_vs_gpu_same_config`` measures both sides on identical small inputs;
``cpu_baseline`` (and ``--impl reference``) is a per-component
extrapolation to the full config, labelled as such.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c3|c2|c1]
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        return float(json.loads(PEAKS.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                r = [c.strip() for c in r]
                util = float(r[6]) if len(r) > 6 and r[6] not in ("", "[N/A]") else 100.0
                if util > 0:
                    sm.append(float(r[0]))
                mx = float(r[1])
                for k, n in enumerate(names):
                    if r[2 + k].lower().startswith("active"):
                        reasons.add(n)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------- CPU oracle
# same-config comparisons: each runs on identical inputs on the GPU (device
# timer) and in the CPU oracle port (oracle/, numpy/SciPy, wall clock)
COMPARE = ("c1", "c3s4", "c4s6")


def _compare_case(name):
    """(model, precompute, initial SystemState, h, description) for a
    same-config comparison. c1 uses the reference's own precompute (bases +
    cubature written by tetsolve, tests/golden/c1.npz); the others the
    injected precompute of the benchmark scenes."""
    from paper_2506_06494_b200 import scenes
    from paper_2506_06494_b200.model import Model, SystemState
    from paper_2506_06494_b200.precompute import Precompute
    if name == "c1":
        with np.load(ROOT / "tests" / "golden" / "c1.npz") as d:
            g = {k: d[k] for k in d.files}
        m = Model.from_arrays(g)
        h = float(g["scene_h"][0])
        st = SystemState(x=g["frame_x_init"][0].copy(), x_prev=g["frame_x_prev"][0].copy(),
                         v=g["frame_v"][0].copy(), z=g["frame_z"][0].copy(), h=h)
        return m, Precompute.from_arrays(g), st, h, "C1 cantilever 10,080 tets, reference precompute"
    m, st, h, desc = scenes.build(name)
    return m, Precompute.injected(m, h, samples=6, seed=0), st, h, desc


def cpu_compare(names=COMPARE, sweeps=2, gpu=True):
    """Measured GPU and CPU-oracle sweeps/s on the same small configs (the
    sizes the reference algorithm can run on a CPU), each from
    the same state for the same ``sweeps`` outer iterations (rotations +
    sweep + tracked energy, local_solver.py:697-716)."""
    from oracle import jgs2_oracle as orc
    from paper_2506_06494_b200.model import SystemState
    out = []
    for name in names:
        m, pre, st, h, desc = _compare_case(name)
        tol = 1e-300  # a fixed number of sweeps
        rec = {"config": name, "workload": desc, "tets": int(m.num_elements), "sweeps": sweeps}
        cp = lambda s: SystemState(x=s.x.copy(), x_prev=s.x_prev.copy(), v=s.v.copy(),  # noqa: E731
                                   z=s.z.copy(), h=s.h)
        solver = orc.OracleSolver(m, pre, h, orc.OracleConfig(max_outer=sweeps, tol_dx=tol))
        s1 = cp(st)
        t0 = time.perf_counter()
        sc = solver.outer_solve(s1)
        t_cpu = time.perf_counter() - t0
        rec["cpu_sweeps_s"] = sc.outer_iterations / t_cpu
        rec["cpu_halvings"] = [int(a) for a in sc.line_search_activations]
        if gpu:
            from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
            g = LocalSolver(m, SolverConfig(max_outer=sweeps, tol_dx=tol), precompute=pre, h_ref=h)
            for rep in range(2):  # warm-up pass, then the timed pass (same start state)
                g.set_state(st.x, st.z, h)
                g.timer_start()
                for _ in range(sweeps):
                    g.sweep_resident(True)
                ms = g.timer_stop()
            xg = g.get_x()
            rec["gpu_sweeps_s"] = sweeps / (ms / 1e3)
            rec["ratio"] = rec["gpu_sweeps_s"] / rec["cpu_sweeps_s"]
            rec["max_rel_dx_vs_oracle"] = float(np.abs(xg - s1.x).max() / max(np.abs(s1.x).max(), 1e-300))
            g.close()
        out.append(rec)
    return out


def cpu_extrapolate(config, budget_s=20.0):
    """Per-component CPU-port model of one sweep at the full ``config``
    (labelled an extrapolation: SURVEY 8(d), the reference cannot run C4's
    brute-force proximity arrays, n_sv x n_st x 3 doubles). Elastic part:
    measured s/tet/sweep on a bounded slice of the same construction without
    contact, times the full element count. Proximity part: measured seconds
    per (surface vertex x surface triangle) test of the reference's
    brute-force find_pairs on the 6-cells/ball tank, times n_sv*n_st of the
    full scene, times the find_pairs calls a productive sweep makes (pairs at
    x, one accepted trial, the tracked energy: local_solver.py:612, 567, 712).
    Returns (s/sweep, components dict)."""
    from oracle import jgs2_oracle as orc
    from paper_2506_06494_b200 import scenes
    from paper_2506_06494_b200.precompute import Precompute
    m_full, _, _, _ = scenes.build(config)
    name = "c1" if config == "c1" else "c3s4"
    m, st, h, _ = scenes.build(name)
    pre = Precompute.injected(m, h, samples=6, seed=0)
    solver = orc.OracleSolver(m, pre, h, orc.OracleConfig(max_outer=1))
    times = []
    t_all = time.perf_counter()
    while len(times) < 3 and time.perf_counter() - t_all < budget_s:
        t0 = time.perf_counter()
        rot = orc.vertex_rotations(m, st.x)
        solver.sweep(st, rot)
        times.append(time.perf_counter() - t0)
    per_tet = statistics.median(times) / m.num_elements
    comp = {"elastic_s_per_sweep": per_tet * m_full.num_elements,
            "elastic_sample": f"{len(times)} oracle sweeps of {name} ({m.num_elements} tets), "
                              f"median {statistics.median(times):.3f} s"}
    total = comp["elastic_s_per_sweep"]
    if m_full.barrier is not None and len(m_full.surface_tris):
        mc, stc, _, _ = scenes.build("c4s6")
        t0 = time.perf_counter()
        orc.find_pairs(mc, stc.x)
        t_fp = time.perf_counter() - t0
        per_test = t_fp / (len(mc.surface_vertices) * len(mc.surface_tris))
        tests = len(m_full.surface_vertices) * len(m_full.surface_tris)
        comp["proximity_s_per_sweep"] = 3 * per_test * tests
        comp["proximity_sample"] = (f"brute-force find_pairs on c4s6 ({len(mc.surface_vertices)} sv x "
                                    f"{len(mc.surface_tris)} st) {t_fp:.3f} s -> {per_test:.3e} s/test; "
                                    f"{tests:.3e} tests x 3 calls per sweep at full size")
        total += comp["proximity_s_per_sweep"]
    comp["extrapolated"] = True
    return total, comp


def traffic(config, kernel, launches, steps):
    """DRAM bytes per launch of the roofline kernel from the committed ncu
    capture (profiles/r2_traffic_<config>.json, else r1_; dram__bytes_read.sum +
    dram__bytes_write.sum summed over the kernel's launches in one sweep),
    or None when no capture exists for this config."""
    try:
        f = ROOT / "profiles" / f"r2_traffic_{config}.json"
        if not f.exists():
            f = ROOT / "profiles" / f"r1_traffic_{config}.json"
        t = json.loads(f.read_text())
        if t.get("phase") != kernel or not launches:
            return None
        return t["dram_bytes_per_sweep"] / (launches / steps)
    except Exception:
        return None


def threads():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    # C4 (3.5M tets, ten puffer balls, IPC) is the configuration BASELINE.json's
    # metric is quoted on; C3 (1M-tet twist, no contact) is the elastic-only case
    ap.add_argument("--config", default=os.environ.get("JGS2_BENCH_CONFIG", "c4"))
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-precompute", action="store_true")
    ap.add_argument("--precompute-sweeps", type=int, default=30)
    args = ap.parse_args()
    from paper_2506_06494_b200 import replicas
    world, rank, local, dist = replicas.setup()
    barrier, max_over_ranks = replicas.barrier, replicas.max_over_ranks
    from paper_2506_06494_b200 import build as _build
    _build.build()  # no-op unless a CUDA source is newer than lib/libjgs2.so
    metric = "JGS2 iterations/sec (sweeps/s) and ms per timestep to residual tol"

    from paper_2506_06494_b200 import scenes
    if args.impl == "reference":
        if rank != 0:
            return
        per, comp = cpu_extrapolate(args.config)
        measured = cpu_compare(gpu=False) if not args.no_cpu else None
        m_full, _, _, desc = scenes.build(args.config)
        v = 1.0 / per
        cores = threads()
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "sweeps/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": 0,
                "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "parallelism": "1 CPU process"},
                "cpu_baseline": {"value": v, "unit": "sweeps/s", "cores": cores, "kind": "port",
                                 "sample": "extrapolated per component (the reference cannot run this "
                                           "config on a CPU): " + json.dumps(comp),
                                 "host": host_info()},
                "measured_small_configs": measured,
                "e2e": {"value": v, "unit": "sweeps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
    from paper_2506_06494_b200.precompute import Precompute
    from paper_2506_06494_b200 import _lib as L
    m, st, h, desc = scenes.build(args.config)
    t0 = time.perf_counter()
    pre = Precompute.injected(m, h, samples=6, seed=0)
    t_pre = time.perf_counter() - t0
    cfg = SolverConfig(max_outer=500, tol_dx=getattr(m, "tol_dx", 1e-3))
    # N > 1: the scene's bodies are split over the ranks (partition.py; one
    # scene, strong scaling) when it has at least N bodies, else replicas
    from paper_2506_06494_b200 import partition
    partitioned = world > 1 and len(partition.body_ranges(m)) >= world
    solver = LocalSolver(m, cfg, precompute=pre, h_ref=h, device=local if world > 1 else 0,
                         dist=dist if partitioned else None, comm="nccl")
    fi = solver.factor_info
    from paper_2506_06494_b200.model import SystemState
    init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
    # the simulation runs on the device: timesteps (compute_z, capped
    # initialize_step, sweeps to tol_dx, velocity update) continue across
    # the warm-up and timed windows; a step is one sweep.
    solver.set_frame_state(init, m.gravity)
    solver.run_sweeps(args.warmup)
    solver.phase_reset()
    solver.profile(True)
    launches0 = solver.kernel_launches
    barrier(dist)
    clocks = Clocks(local)
    record = []
    solver.timer_start()
    frames_done = solver.run_sweeps(args.steps, record)
    ms = solver.timer_stop()
    barrier(dist)
    clk = clocks.stop()
    launches = solver.kernel_launches - launches0
    ms = max_over_ranks(dist, ms)
    phases = solver.phase_stats()
    solver.profile(False)
    # partitioned: every rank advanced the same scene by args.steps sweeps
    value = (args.steps / (ms / 1e3) if partitioned else replicas.job_throughput(dist, args.steps, ms / 1e3))
    hv = np.array([r["halvings"] for r in record])
    mh = cfg.max_halvings
    accepted = hv <= mh
    sweeps_info = {
        "halvings_hist": {str(k): int(c) for k, c in zip(*np.unique(hv, return_counts=True))},
        "frac_le5_halvings": float(np.mean(hv <= 5)),
        "floored": int(np.sum(~accepted)),
        "mean_gamma_over_cap_accepted": (float(np.mean([r["gamma"] / r["cap"] for r, a in zip(record, accepted)
                                                        if a and r["cap"] > 0])) if accepted.any() else None),
        "mean_pairs": float(np.mean([r["n_pairs"] for r in record])),
        "mean_indefinite_elements": float(np.mean([r["n_indefinite"] for r in record])),
    }

    # roofline of the dominant HBM-modelled kernel (3x3-block arithmetic +
    # sparse triangular solves; the contact phases are latency/search bound
    # and carry no algorithmic bytes in the SURVEY 8(d) model)
    peak, peak_kind = hbm_peak()
    dom = max((p for p in phases if phases[p][2] > 0), key=lambda p: phases[p][0])
    d_ms, d_launch, d_bytes = phases[dom]
    achieved = d_bytes / (d_ms / 1e3) / 1e9 if d_ms > 0 else 0.0
    total_bytes = sum(p[2] for p in phases.values())
    # the same kernel without the element Hessians running beside it (they
    # share its SMs in the timed window): a short untimed window after it
    standalone = None
    if dom == "factor_solve" and args.steps > 0:
        solver.set_hess_overlap(0)
        solver.phase_reset()
        solver.profile(True)
        solver.run_sweeps(min(args.steps, 10))
        s_ms, s_launch, s_bytes = solver.phase_stats()[dom]
        solver.profile(False)
        solver.set_hess_overlap(1)
        if s_ms > 0:
            s_ach = s_bytes / (s_ms / 1e3) / 1e9
            standalone = {"achieved": s_ach, "frac": s_ach / peak, "ms_per_step": s_ms / min(args.steps, 10),
                          "sweeps": min(args.steps, 10),
                          "note": "element Hessians before the local systems instead of under the solve"}

    # whole timesteps to the residual tolerance, device-resident: close the
    # frame left open by the window (untimed), then time complete frames
    if getattr(solver, "_frame_open", False):
        while getattr(solver, "_frame_open", False):
            solver.run_sweeps(1)
    ts = []
    for _ in range(args.frames):
        solver.timer_start()
        (it, conv), = solver.run_frames(1)
        ts.append((it, conv, solver.timer_stop()))

    # end-to-end through the public API with HOST buffers: one
    # LocalSolver.timestep call per frame (jgs2_timestep_host: the frame
    # state x_prev, v goes h2d from pinned host memory, compute_z + capped
    # initialize_step + outer_solve to tol_dx + velocity update run on the
    # device, the new x_prev, v come back d2h), from the scene's initial
    # state over whole frames covering at least the timed window's sweeps
    # (the same frames the device-resident window ran)
    nv = m.num_vertices
    xpw, o7 = L.pinned_array((nv, 3))
    vvw, o8 = L.pinned_array((nv, 3))
    xpw[:], vvw[:] = init.x_prev, init.v
    e2e_sweeps, e2e_frames, h2d, d2h = 0, 0, 0, 0
    t_e2e = time.perf_counter()
    e2e_target = args.e2e_steps if args.e2e_steps is not None else args.warmup + args.steps
    while e2e_sweeps < e2e_target:
        fs = SystemState(x=None, x_prev=xpw, v=vvw, z=None, h=h)
        it, _ = solver.timestep(fs, m.gravity, x_prev_out=xpw, v_out=vvw)
        h2d += 2 * xpw.nbytes
        d2h += 2 * xpw.nbytes
        e2e_sweeps += it
        e2e_frames += 1
    e2e_s = time.perf_counter() - t_e2e
    e2e = (e2e_sweeps / replicas.max_over_ranks(dist, e2e_s) if partitioned
           else replicas.job_throughput(dist, e2e_sweeps, e2e_s))

    fill = None
    if rank == 0:
        try:
            t0 = time.perf_counter()
            stored, own_exact, metis = solver.factor_fill()
            fill = {"nnz_L_stored": stored, "nnz_L_exact_this_ordering": own_exact,
                    "nnz_L_exact_metis_whole_graph": metis, "stored_over_metis": stored / metis,
                    "seconds": round(time.perf_counter() - t0, 1)}
        except Exception as exc:
            fill = {"failed": str(exc)}

    # the scalable precompute at this config, and sweeps driven
    # by it: the reference algorithm's own bases/cubature instead of the
    # injected ones (rank 0 only, after the timed windows)
    scal = None
    if rank == 0 and not args.no_precompute:
        solver.close()
        try:
            scal = scalable_block(m, h, cfg, init, args.precompute_sweeps)
        except Exception as exc:  # never fail the GPU line on this block
            scal = {"failed": str(exc)}

    cpu, compare = None, None
    if rank == 0 and not args.no_cpu:
        try:
            per, comp = cpu_extrapolate(args.config)
            cpu = {"value": 1.0 / per, "unit": "sweeps/s", "cores": threads(), "kind": "port",
                   "sample": "extrapolated per component: " + json.dumps(comp), "host": host_info()}
        except Exception as exc:  # never fail the GPU line on the CPU sample
            cpu = {"value": None, "unit": "sweeps/s", "cores": threads(), "kind": "port",
                   "sample": f"failed: {exc}"}
        try:
            compare = cpu_compare()
        except Exception as exc:
            compare = [{"failed": str(exc)}]
    if rank != 0:
        return
    line = {
        "metric": metric, "value": value, "unit": "sweeps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if partitioned else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "tets": m.num_elements, "vertices": nv,
                   "precompute": "injected (structurally valid; Precompute.injected)",
                   "cubature_samples": 6, "h": h, "tol_dx": cfg.tol_dx,
                   "parallelism": (f"body partition x{world} (rank 0 vertices {solver.partition})" if partitioned
                                   else f"replicas x{world}"),
                   "l2": "inputs > L2 (factor %.2f GB)" % (8 * fi.nnz_dof / 1e9)},
        "sweeps": sweeps_info,
        "timestep": {"frames": [{"sweeps": it, "converged": cv, "ms": round(t, 2)} for it, cv, t in ts],
                     "ms_per_timestep": float(np.mean([t for _, _, t in ts])) if ts else None,
                     "mean_sweeps_per_frame": float(np.mean([it for it, _, _ in ts])) if ts else None,
                     "frames_completed_in_window": frames_done},
        "factor": {"nnz_L": int(fi.nnz_dof), "fronts": int(fi.nfronts), "levels": int(fi.nlevels),
                   "max_front": int(fi.max_front),
                   "ordering": "METIS nested dissection" if fi.ordering == 1 else "geometric nested dissection",
                   "fill_vs_metis": fill,
                   "factor_s": round(solver.factor_seconds, 2), "precompute_s": round(t_pre, 2)},
        "roofline": {"bound": "hbm", "kernel": dom,
                     "dominant_phase": max(phases, key=lambda p: phases[p][0]), "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic(args.config, dom, d_launch, args.steps),
                     "bytes_per_launch": d_bytes / max(d_launch, 1), "launches": d_launch,
                     "step_bytes": total_bytes / args.steps,
                     "step_frac": (total_bytes / (ms / 1e3) / 1e9) / peak,
                     "in_step": "timed window: the element Hessians share the SMs with the solve",
                     "standalone": standalone},
        "phases_ms_per_step": {p: round(v[0] / args.steps, 4) for p, v in phases.items()},
        "phases_gbs": {p: round(v[2] / (v[0] / 1e3) / 1e9, 1) for p, v in phases.items()
                       if v[0] > 0 and v[2] > 0},
        "e2e": {"value": e2e, "unit": "sweeps/s", "h2d_bytes_per_step": h2d / max(e2e_sweeps, 1),
                "d2h_bytes_per_step": d2h / max(e2e_sweeps, 1), "sweeps": e2e_sweeps, "frames": e2e_frames,
                "timing": "wall clock: one LocalSolver.timestep (jgs2_timestep_host) per frame: "
                          "x_prev, v h2d from pinned host memory, compute_z + capped initialize_step "
                          "+ outer_solve to tol_dx + velocity update on the device, x_prev, v d2h"},
        "gpu_launches": launches,
        "host_rss_gb": round(__import__("resource").getrusage(__import__("resource").RUSAGE_SELF).ru_maxrss / 2**20, 2),
        "clocks": clk,
        "cpu_baseline": cpu,
        "cpu_vs_gpu_same_config": compare,
        "precompute_scalable": scal,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def scalable_block(m, h, cfg, init, sweeps):
    """Device precompute of the scene (precompute_gpu.py) and ``sweeps``
    sweeps of the continuing simulation driven by it."""
    from paper_2506_06494_b200.local_solver import LocalSolver
    from paper_2506_06494_b200.precompute_gpu import scalable_precompute
    t0 = time.perf_counter()
    pre, info = scalable_precompute(m, h)
    out = {"seconds": round(time.perf_counter() - t0, 2)}
    res = info.pop("residual")
    info.pop("converged")
    out.update({k: (round(v, 4) if isinstance(v, float) else v) for k, v in info.items()})
    out["residual_p90"] = float(np.quantile(res, 0.9)) if res.size else 0.0
    s = LocalSolver(m, cfg, precompute=pre, h_ref=h)
    s.set_frame_state(init, m.gravity)
    s.run_sweeps(2)
    rec = []
    s.timer_start()
    frames = s.run_sweeps(sweeps, rec)
    ms = s.timer_stop()
    hv = np.array([r["halvings"] for r in rec])
    out.update({"sweeps_s": sweeps / (ms / 1e3), "sweeps": sweeps, "frames_completed": frames,
                "halvings_hist": {str(k): int(c) for k, c in zip(*np.unique(hv, return_counts=True))},
                "frac_le5_halvings": float(np.mean(hv <= 5)), "floored": int(np.sum(hv > cfg.max_halvings))})
    s.close()
    return out


def host_info():
    """CPU model, threads and the numpy/SciPy/BLAS stack."""
    info = {"nproc": os.cpu_count()}
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                info["cpu"] = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        import scipy
        info["numpy"], info["scipy"] = np.__version__, scipy.__version__
        import threadpoolctl
        info["blas"] = [{k: i.get(k) for k in ("internal_api", "version", "num_threads")}
                        for i in threadpoolctl.threadpool_info()]
    except Exception:
        pass
    info["OMP_NUM_THREADS"] = os.environ.get("OMP_NUM_THREADS")
    return info


if __name__ == "__main__":
    main()
