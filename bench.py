"""Benchmark of the JGS2 runtime iteration on B200 (driver contract).

A *step* is one JGS2 outer iteration (Jacobi sweep in corotated_cubature
mode incl. rotation refresh, exact reduced collect, sampled corrections,
local line search and the sweep-level backtracking guard), i.e. one
``LocalSolver.outer_solve`` iteration (reference local_solver.py:697-716).
``value`` = sweeps/s over all ranks with the state resident in HBM;
``e2e`` = the same through the C-ABI host-buffer call (x, z in from pinned
host memory, x, dx out, every step). ``--impl reference`` times the CPU
oracle port of the reference (numpy/SciPy, oracle/) on a bounded sample.

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
def cpu_sample(config, steps=3, budget_s=25.0):
    """Time the CPU oracle port (oracle/jgs2_oracle.py) on a bounded sample
    of the workload and extrapolate to the full scene; returns (seconds per
    sweep at full size, description).

    * elastic sweep: the same construction scaled down to ~10K tets
      (injected precompute), ``steps`` sweeps, median s/sweep scaled linearly
      in element count (84-89 us/tet/sweep is linear in ne);
    * contact scenes (the reference's brute-force proximity
      needs n_sv x n_st x 3 doubles at C4, petabytes, so it is not runnable):
      one brute-force find_pairs on the 10-body scene at 6 cells/ball, scaled
      by n_sv * n_st, times the 3 calls a sweep makes at least (pairs at x,
      one backtracking trial, the tracked energy; local_solver.py:612, 567,
      712) -- a lower bound on the reference's contact cost.
    """
    from oracle import jgs2_oracle as orc
    from paper_2506_06494_b200 import scenes
    from paper_2506_06494_b200.precompute import Precompute
    m_full, _, _, _ = scenes.build(config)
    name = "c1" if config == "c1" else "c3s4"
    m, st, h, _ = scenes.build(name)
    pre = Precompute.injected(m, h, samples=6, seed=0)
    solver = orc.OracleSolver(m, pre, h, orc.OracleConfig(max_outer=steps))
    times = []
    t_all = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        rot = orc.vertex_rotations(m, st.x)
        solver.sweep(st, rot)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s:
            break
    per_tet = statistics.median(times) / m.num_elements
    per_sweep = per_tet * m_full.num_elements
    desc = (f"oracle port: {len(times)} sweeps of {name} ({m.num_elements} tets, injected precompute), "
            f"median s/sweep scaled linearly by element count to {m_full.num_elements} tets")
    if m_full.barrier is not None and len(m_full.surface_tris):
        mc, stc, _, _ = scenes.build("c4s6")
        t0 = time.perf_counter()
        orc.find_pairs(mc, stc.x)
        t_fp = time.perf_counter() - t0
        scale = (len(m_full.surface_vertices) * len(m_full.surface_tris)) / (
            len(mc.surface_vertices) * len(mc.surface_tris))
        per_sweep += 3 * t_fp * scale
        desc += (f" + 3 brute-force find_pairs per sweep: one call on c4s6 ({len(mc.surface_vertices)} sv x "
                 f"{len(mc.surface_tris)} st) took {t_fp:.2f} s, scaled by n_sv*n_st x{scale:.0f} "
                 f"(extrapolation; the reference cannot run C4's proximity arrays)")
    return per_sweep, desc


def traffic(config, kernel, launches, steps):
    """DRAM bytes per launch of the roofline kernel from the committed ncu
    capture (profiles/r1_traffic_<config>.json, dram__bytes_read.sum +
    dram__bytes_write.sum summed over the kernel's launches in one sweep),
    or None when no capture exists for this config."""
    try:
        t = json.loads((ROOT / "profiles" / f"r1_traffic_{config}.json").read_text())
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
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    # C4 (3.5M tets, ten puffer balls, IPC) is the configuration BASELINE.json's
    # metric is quoted on; C3 (1M-tet twist, no contact) is the elastic-only case
    ap.add_argument("--config", default=os.environ.get("JGS2_BENCH_CONFIG", "c4"))
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu", action="store_true")
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
        per, sample = cpu_sample(args.config, steps=max(min(args.steps, 3), 1))
        m_full, _, _, desc = scenes.build(args.config)
        v = 1.0 / per
        cores = threads()
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "sweeps/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": 0,
                "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "parallelism": "1 CPU process"},
                "cpu_baseline": {"value": v, "unit": "sweeps/s", "cores": cores, "kind": "port",
                                 "sample": sample},
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
    solver = LocalSolver(m, cfg, precompute=pre, h_ref=h, device=local if world > 1 else 0)
    fi = solver.factor_info
    from paper_2506_06494_b200.model import SystemState
    init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
    # the simulation runs on the device: timesteps (compute_z, capped
    # initialize_step, sweeps to tol_dx, velocity update) continue across
    # the warm-up and timed windows; a step is one sweep.
    solver.set_frame_state(init, m.gravity)
    episode = getattr(m, "episode_frames", None)
    solver.run_sweeps(args.warmup, episode)
    solver.phase_reset()
    solver.profile(True)
    launches0 = solver.kernel_launches
    barrier(dist)
    clocks = Clocks(local)
    solver.timer_start()
    frames_done = solver.run_sweeps(args.steps, episode)
    ms = solver.timer_stop()
    barrier(dist)
    clk = clocks.stop()
    launches = solver.kernel_launches - launches0
    ms = max_over_ranks(dist, ms)
    phases = solver.phase_stats()
    solver.profile(False)
    value = replicas.job_throughput(dist, args.steps, ms / 1e3)

    # roofline of the dominant HBM-modelled kernel (3x3-block arithmetic +
    # sparse triangular solves; the contact phases are latency/search bound
    # and carry no algorithmic bytes in the SURVEY 8(d) model)
    peak, peak_kind = hbm_peak()
    dom = max((p for p in phases if phases[p][2] > 0), key=lambda p: phases[p][0])
    d_ms, d_launch, d_bytes = phases[dom]
    achieved = d_bytes / (d_ms / 1e3) / 1e9 if d_ms > 0 else 0.0
    total_bytes = sum(p[2] for p in phases.values())

    # one full timestep to the residual tolerance, device-resident
    solver.timer_start()
    (ts_iters, ts_conv), = solver.run_frames(1)
    ts_ms = solver.timer_stop()

    # end-to-end through the public API with HOST buffers: one
    # LocalSolver.timestep call per frame (jgs2_timestep_host: the frame
    # state x_prev, v goes h2d from pinned host memory, compute_z + capped
    # initialize_step + outer_solve to tol_dx + velocity update run on the
    # device, the new x_prev, v come back d2h), the same episode resets as
    # the timed window (an episode's first frame reads the initial state)
    import ctypes
    nv = m.num_vertices
    xp0, o5 = L.pinned_array((nv, 3))
    vv0, o6 = L.pinned_array((nv, 3))
    xpw, o7 = L.pinned_array((nv, 3))
    vvw, o8 = L.pinned_array((nv, 3))
    xp0[:], vv0[:] = init.x_prev, init.v
    e2e_sweeps, e2e_frames, h2d, d2h = 0, 0, 0, 0
    t_e2e = time.perf_counter()
    while e2e_sweeps < args.e2e_steps:
        first = e2e_frames == 0 or bool(episode and e2e_frames % episode == 0)
        fs = SystemState(x=None, x_prev=xp0 if first else xpw, v=vv0 if first else vvw, z=None, h=h)
        it, _ = solver.timestep(fs, m.gravity, x_prev_out=xpw, v_out=vvw)
        h2d += 2 * xpw.nbytes
        d2h += 2 * xpw.nbytes
        e2e_sweeps += it
        e2e_frames += 1
    e2e = replicas.job_throughput(dist, e2e_sweeps, time.perf_counter() - t_e2e)
    e2e_h2d, e2e_d2h, e2e_n, e2e_f = h2d, d2h, e2e_sweeps, e2e_frames

    # secondary: the reference harness's own loop around the drop-in
    # LocalSolver (harness.py run loop): per frame host
    # compute_z, initialize_step (feasibility cap through the ABI), then
    # LocalSolver.outer_solve(state) -- x, z uploaded from pinned host memory,
    # sweeps to tol_dx, x and the rotations read back into pinned memory --
    # and the host velocity update (in place on preallocated arrays); the same
    # episode resets as the timed window
    px, o1 = L.pinned_array((nv, 3))
    pz, o2 = L.pinned_array((nv, 3))
    pdz, o3 = L.pinned_array((nv, 3))
    prot, o4 = L.pinned_array((nv, 9))
    # from the scene's initial state, like every episode of the timed window
    xp0, vv0 = np.array(init.x_prev, dtype=np.float64), np.array(init.v, dtype=np.float64)
    xprev, vel = xp0.copy(), vv0.copy()           # host frame state
    grav = (h * h) * np.asarray(m.gravity, dtype=np.float64)
    fixed = np.flatnonzero(np.asarray(m.fixed_mask))
    inf = L.SweepInfo()
    lib, ctx = solver._lib, solver._ctx
    cap_d = L.f64(1.0)
    e2e_sweeps, e2e_frames, h2d, d2h = 0, 0, 0, 0
    tdbg = {} if os.environ.get("JGS2_E2E_DEBUG") else None

    def mark(key, t0):
        if tdbg is not None:
            tdbg[key] = tdbg.get(key, 0.0) + time.perf_counter() - t0
            tdbg.setdefault(key + "_list", []).append(round(1e3 * (time.perf_counter() - t0), 2))
        return time.perf_counter()
    t_e2e = time.perf_counter()
    while e2e_sweeps < args.e2e_steps:
        if episode and e2e_frames and e2e_frames % episode == 0:
            xprev[:], vel[:] = xp0, vv0
        t0 = time.perf_counter()
        np.multiply(vel, h, out=pz)                  # compute_z (assembly.py:165-180), in place
        pz += xprev
        pz += grav
        pz[fixed] = xprev[fixed]
        np.subtract(pz, xprev, out=pdz)
        px[:] = xprev
        t0 = mark("host_z", t0)
        L.check(lib.jgs2_step_cap(ctx, L.ptr(px, L.f64), L.ptr(pdz, L.f64), ctypes.byref(cap_d)), ctx)
        t0 = mark("step_cap", t0)
        pdz *= cap_d.value                           # initialize_step (harness.py:130-134)
        px += pdz
        L.check(lib.jgs2_set_state(ctx, L.ptr(px, L.f64), L.ptr(pz, L.f64), h), ctx)
        h2d += 4 * px.nbytes
        t0 = mark("set_state", t0)
        for it in range(cfg.max_outer):              # outer_solve (local_solver.py:688-721)
            L.check(lib.jgs2_sweep(ctx, 1, ctypes.byref(inf)), ctx)
            e2e_sweeps += 1
            if inf.dx_norm < cfg.tol_dx:
                break
        t0 = mark("sweeps", t0)
        L.check(lib.jgs2_get_x(ctx, L.ptr(px, L.f64)), ctx)
        L.check(lib.jgs2_get_rotations(ctx, L.ptr(prot, L.f64)), ctx)
        d2h += px.nbytes + prot.nbytes
        t0 = mark("readback", t0)
        np.subtract(px, xprev, out=vel)              # step_velocity_update (assembly.py:346-351)
        vel *= 1.0 / h
        xprev[:] = px
        t0 = mark("host_v", t0)
        e2e_frames += 1
    e2e_h = replicas.job_throughput(dist, e2e_sweeps, time.perf_counter() - t_e2e)
    if tdbg is not None:
        print("e2e breakdown (s):", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in tdbg.items()},
              file=sys.stderr)

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            per, sample = cpu_sample(args.config)
            cpu = {"value": 1.0 / per, "unit": "sweeps/s", "cores": threads(), "kind": "port",
                   "sample": sample}
        except Exception as exc:  # never fail the GPU line on the CPU sample
            cpu = {"value": None, "unit": "sweeps/s", "cores": threads(), "kind": "port",
                   "sample": f"failed: {exc}"}
    if rank != 0:
        return
    line = {
        "metric": metric, "value": value, "unit": "sweeps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "tets": m.num_elements, "vertices": nv,
                   "precompute": "injected (structurally valid; Precompute.injected)",
                   "cubature_samples": 6, "h": h, "parallelism": f"replicas x{world}",
                   "l2": "inputs > L2 (factor %.2f GB)" % (8 * fi.nnz_dof / 1e9)},
        "episode_frames": episode,
        "timestep": {"iterations": ts_iters, "converged": ts_conv, "ms": ts_ms,
                     "frames_in_window": len(frames_done),
                     "mean_sweeps_per_frame": (float(np.mean(frames_done)) if frames_done else None),
                     "ms_per_timestep": (ms / args.steps * float(np.mean(frames_done))
                                         if frames_done else None)},
        "factor": {"nnz_L": int(fi.nnz_dof), "fronts": int(fi.nfronts), "levels": int(fi.nlevels),
                   "max_front": int(fi.max_front), "ordering": "geometric nested dissection",
                   "factor_s": round(solver.factor_seconds, 2), "precompute_s": round(t_pre, 2)},
        "roofline": {"bound": "hbm", "kernel": dom,
                     "dominant_phase": max(phases, key=lambda p: phases[p][0]), "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic(args.config, dom, d_launch, args.steps),
                     "bytes_per_launch": d_bytes / max(d_launch, 1), "launches": d_launch,
                     "step_bytes": total_bytes / args.steps,
                     "step_frac": (total_bytes / (ms / 1e3) / 1e9) / peak},
        "phases_ms_per_step": {p: round(v[0] / args.steps, 4) for p, v in phases.items()},
        "phases_gbs": {p: round(v[2] / (v[0] / 1e3) / 1e9, 1) for p, v in phases.items()
                       if v[0] > 0 and v[2] > 0},
        "e2e": {"value": e2e, "unit": "sweeps/s", "h2d_bytes_per_step": e2e_h2d / max(e2e_n, 1),
                "d2h_bytes_per_step": e2e_d2h / max(e2e_n, 1), "sweeps": e2e_n, "frames": e2e_f,
                "timing": "wall clock: one LocalSolver.timestep (jgs2_timestep_host) per frame: "
                          "x_prev, v h2d from pinned host memory, compute_z + capped initialize_step "
                          "+ outer_solve to tol_dx + velocity update on the device, x_prev, v d2h"},
        "e2e_harness_loop": {"value": e2e_h, "unit": "sweeps/s", "h2d_bytes_per_step": h2d / max(e2e_sweeps, 1),
                             "d2h_bytes_per_step": d2h / max(e2e_sweeps, 1), "sweeps": e2e_sweeps,
                             "frames": e2e_frames,
                             "timing": "wall clock: the reference harness loop around the drop-in: per frame "
                                       "host numpy compute_z + capped initialize_step + outer_solve(state) from "
                                       "pinned host x, z (x, rotations read back) + host numpy velocity update"},
        "gpu_launches": launches,
        "host_rss_gb": round(__import__("resource").getrusage(__import__("resource").RUSAGE_SELF).ru_maxrss / 2**20, 2),
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
