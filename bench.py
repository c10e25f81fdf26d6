"""Benchmark of the B200 sliding-mesh DG right-hand side + RK step.

Workload (BASELINE.json configs[4], the largest configuration the reference's
algorithm covers on one GPU — configs[1]-[3] need non-matching / oblique /
curved / rotating interfaces that neither the reference nor this round
implements): Taylor-Green vortex in [0, 2pi]^3 at M=0.1,
Re=1600, three blocks stacked along BASELINE z with two planar sliding
interfaces at 2pi/3 and 4pi/3, middle block sliding at +0.2 along BASELINE x;
64^3 elements per GPU, N=5 Gauss nodes, fp64, viscous.  One "step" = one
5-stage low-storage RK step (5 right-hand sides + mortars + updates).

metric: DOF-updates/s = E*(N+1)^3 * 5 * steps / time, whole job over all GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import glob
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

import numpy as np  # noqa: E402

METRIC = "DOF-updates/s (1/PID) per GPU, DG RHS+sliding mortars, 1/2/4/8 B200"
UNIT = "DOF-updates/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--degree", type=int, default=5)
    p.add_argument("--elems", type=int, default=64, help="elements per direction per GPU (weak scaling)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--mesh", default="tgv", choices=["tgv", "warped", "rotor"],
                   help="tgv: affine hexahedra (configs[4]); warped: the same case on curved hexahedra "
                        "(SDG_MAP_WARP, amplitude 5%% of the element size as in configs[3]); rotor: configs[3], "
                        "1.1M-element stator/rotor/stator 20-degree annulus sector (SDG_MAP_ANNULUS), strong scaling")
    return p.parse_args()


def tgv_mesh(T, elems_x, elems_yz, warp=None, copies=1):
    """Three blocks along x (= BASELINE z); interfaces at 2pi/3, 4pi/3.  Weak scaling over
    `copies` GPUs stacks that many periods of the (2 pi periodic) TGV along the sliding
    direction y and splits it in y slabs through all three blocks (partition 2): every GPU
    holds one identical 64^3 TGV box, both sliding interfaces included."""
    L = 2.0 * math.pi
    base, rem = divmod(elems_x, 3)
    n = [base + (rem == 2), base + (rem == 1), base + (rem == 2)]
    bands = [(n[0], 1.0, 0.0), (n[1], 1.0, 0.2), (n[2], 1.0, 0.0)]
    return T.mesh_spec(bands, ny=elems_yz * copies, nz=elems_yz, width=L, height=L * copies, depth=L, warp=warp,
                       partition=T.PARTITION_YSLAB if copies > 1 else T.PARTITION_LEX), bands


WARP = 0.05  # BASELINE configs[3]: "sinusoidal mesh warping of amplitude 5% of element size"


def rotor_workload(args, world, elements=None):
    """BASELINE configs[3] (turbine-scale synthetic): three axial blocks (stator,
    rotor, stator) of a 20-degree periodic annulus sector r in [0.8, 1] with two
    sliding interfaces, 5% warping inside the blocks (x and r), tip Mach 0.4,
    axial inflow M = 0.3 (density-wave perturbation 1e-2), Re = 8e5 on the
    mean-radius arc of the sector, N = 5.  About 1.1M curved hexahedra in total
    (192 axial x 96 around x 60 radial), partitioned over the GPUs (strong
    scaling).  `elements` = (nx, n_theta, n_r) overrides the mesh (CPU sample)."""
    from paper_2008_04356_b200 import types as T
    gamma, mach, rho0, u0 = 1.4, 0.3, 2.0, 1.0
    p0 = rho0 * u0 * u0 / (gamma * mach * mach)
    c0 = math.sqrt(gamma * p0 / rho0)
    r_in, r_out = 0.8, 1.0
    omega = 0.4 * c0 / r_out
    span = math.pi / 9.0
    chord = 0.5 * (r_in + r_out) * span
    mu = rho0 * u0 * chord / 8e5
    nx, n_theta, n_r = elements or (192, 96, 60)
    base, rem = divmod(nx, 3)
    n = [base + (rem == 2), base + (rem == 1), base + (rem == 2)]
    bands = [(n[0], 1.0, 0.0), (n[1], 1.0, omega), (n[2], 1.0, 0.0)]
    mesh = T.annulus_spec(bands, n_theta, n_r, r_in, r_out, length=1.0, warp=WARP, theta_span=span)
    cfg = T.solver_config(args.degree, T.NODES_GAUSS, gamma=gamma, R=1.0, mu=mu, Pr=0.72,
                          case=T.density_wave(alpha=0.02, a=(u0, 0.0, 0.0), k=(2.0, 0.0, 0.0), p0=p0))
    n1 = args.degree + 1
    E = nx * n_theta * n_r
    conf = {
        "workload": f"BASELINE configs[3]: stator/rotor/stator annulus sector r in [{r_in}, {r_out}], 20 degrees "
                    f"(rotationally periodic), 2 sliding interfaces, rotor omega {omega:.4f} (tip Mach 0.4), "
                    f"warp {WARP}, axial M=0.3 inflow with 1e-2 density perturbation, Re=8e5, "
                    f"{nx}x{n_theta}x{n_r} = {E} curved hexahedra over {world} GPU(s), N={args.degree} Gauss, viscous",
        "geometry": "curved",
        "elements": E,
        "elements_per_gpu": E // world,
        "degree": args.degree,
        "nodes": "gauss",
        "dof": E * n1 ** 3,
        "bands_nx": n,
        "l2_policy": "inputs larger than L2 (state %.0f MB per GPU)" % (E // world * n1 ** 3 * 40 / 1e6),
        "parallelism": f"dp{world} (element partition, NCCL halo + mortar exchange)",
        "scaling": "strong",
    }
    return mesh, cfg, conf, E * n1 ** 3


def workload(args, world):
    from paper_2008_04356_b200 import types as T
    if args.mesh == "rotor":
        return rotor_workload(args, world)
    curved = args.mesh == "warped"
    mesh, bands = tgv_mesh(T, args.elems, args.elems, warp=WARP if curved else None, copies=world)
    cfg = T.solver_config(args.degree, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1.0 / 1600.0, Pr=0.72, case=T.tgv())
    n1 = args.degree + 1
    E = sum(b[0] for b in bands) * args.elems * args.elems * world
    geom = (f"curved hexahedra (SDG_MAP_WARP, warp {WARP} of the element size, as BASELINE configs[3]; "
            f"per-node metrics)" if curved else "affine hexahedra")
    conf = {
        "workload": f"BASELINE configs[4]: TGV M=0.1 Re=1600, 3 blocks, 2 planar sliding interfaces (middle +0.2), "
                    f"{args.elems}^3 elements/GPU, N={args.degree} Gauss, viscous, {geom}",
        "geometry": "curved" if curved else "affine",
        "elements": E,
        "elements_per_gpu": E // world,
        "degree": args.degree,
        "nodes": "gauss",
        "dof": E * n1 ** 3,
        "bands_nx": [b[0] for b in bands],
        "l2_policy": "inputs larger than L2 (state %.0f MB, face traces %.0f MB per GPU)" % (
            E // world * n1 ** 3 * 40 / 1e6, E // world * 6 * n1 ** 2 * 72 / 1e6),
        "parallelism": (f"dp{world} (y slabs through all three blocks, NCCL halo + mortar exchange)" if world > 1 else "dp1"),
    }
    return mesh, cfg, conf, E * n1 ** 3


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(args, conf, timeout_s=20.0):
    """The 3D CPU oracle (restatement of the reference path, 'port') on a bounded
    sample of the same workload: same case/degree, reduced mesh, all host threads."""
    from oracle import pyoracle as P
    from paper_2008_04356_b200 import types as T
    threads = os.cpu_count() or 1
    P.oracle_lib().orc_set_threads(threads)
    e = 6
    curved = conf.get("geometry") == "curved"
    if args.mesh == "rotor":
        mesh, cfg, _, _ = rotor_workload(args, 1, elements=(9, 12, 4))
        e = "9x12x4"
    else:
        mesh, bands = tgv_mesh(T, e, e, warp=WARP if curved else None)
        cfg = T.solver_config(args.degree, T.NODES_GAUSS, mu=1.0 / 1600.0, case=T.tgv())
    o = P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    # A timing sample, not a simulation: a small fixed step (well inside the CFL limit) keeps
    # the coarse sample admissible for the whole window (an under-resolved TGV at CFL 0.5
    # leaves the admissible set after ~1000 steps).
    dt = min(1e-3, 0.25 * o.suggest_dt(1.0))
    o.step(dt, 1)  # warm-up
    steps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < timeout_s or steps == 0:
        try:
            o.step(dt, 1)
        except P.T.InvalidStateError if hasattr(P, "T") else Exception:
            if steps == 0:
                raise
            break
        steps += 1
    el = time.perf_counter() - t0
    dof = o.n_elements * (args.degree + 1) ** 3
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    out = {"value": dof * 5 * steps / el, "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"oracle/sdg3d.cpp (OpenMP, {threads} threads, {model}) on the same "
                     f"{'rotor annulus' if args.mesh == 'rotor' else 'TGV'} case"
                     f"{' (curved)' if curved else ''} at {e if isinstance(e, str) else f'{e}^3'} elements (N={args.degree}, {dof} DOF), {steps} RK steps in {el:.1f} s"}
    try:
        out["reference_2d"] = reference_2d(args.degree, seconds=min(8.0, timeout_s))
    except Exception as ex:  # supplementary: never fail the bench line over it
        out["reference_2d"] = {"unavailable": str(ex)[:200]}
    return out


def reference_2d(degree, seconds=8.0):
    """the UNMODIFIED reference library (oracle/_ref, compiled from
    /root/reference/proj/src) on the 2D analog of configs[4]: 3 bands with the
    middle one sliding at 0.2, viscous (mu = 1/1600), Gauss nodes, 48 x 48
    elements (the reference has no TGV case; its density wave stands in), run by
    the reference's own runner with one thread per rank (Backend::InProc).
    Supplementary only: a 2D node carries 4 variables and 2 directions of work."""
    from oracle import pyoracle as P
    if not os.path.exists(P.REF_SO):
        return {"unavailable": "oracle/_ref/libsdg_ref.so not built"}
    ranks = max(3, min(os.cpu_count() or 1, 48))
    spec = P.ref_spec([(16, 1.0, 0.0), (16, 1.0, 0.2), (16, 1.0, 0.0)], 48, degree, mu=1.0 / 1600.0)
    ref = P.Ref2D(spec)
    dt = 0.5 * ref.suggest_dt(0.5)
    _, w = ref.run(dt, 2, ranks=ranks)
    n = max(2, int(seconds / max(w / 2, 1e-6)))
    _, wall = ref.run(dt, n, ranks=ranks)
    nodes = 48 * 48 * (degree + 1) ** 2
    return {"value": nodes * 5 * n / wall, "unit": "2D node-stage-updates/s", "ranks": ranks, "kind": "reference",
            "sample": f"reference runner (InProc threads, {ranks} ranks), 2D 48x48 elements, N={degree} Gauss, "
                      f"viscous, 3 bands, {n} RK steps in {wall:.1f} s (stepping-loop wall, runner.cpp:41-43)"}


def reference_arm(args, world, rank):
    """--impl reference: the CPU implementation of the path on the host cores.
    The reference library itself is 2D-only, so the 3D restatement
    of its algorithm (oracle/sdg3d.cpp, 'port') runs this arm."""
    if rank != 0:
        return
    mesh, cfg, conf, dof = workload(args, 1)
    base = cpu_baseline(args, conf, timeout_s=max(2.0, 3.0 * args.steps / max(args.steps + args.warmup, 1)))
    line = {"metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": conf.get("scaling", "weak"),
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (TGV initial field, analytic)",
            "config": conf, "impl": "reference", "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def b_flow(degree, curved=False):
    """algorithmic bytes per DOF-update of the reference's
    five-pass phase structure (the contract figure)."""
    n1 = degree + 1
    return (400 + 2904 / n1) if curved else (240 + 2712 / n1)


def roofline(kt, conf, args, peaks, value_per_gpu, ms_per_step):
    """Contract roofline: achieved = DOF-updates/s x B_flow, over the
    RK stage (the two fused element kernels + mortar kernels).  Per-kernel
    numbers of this implementation's own fused dataflow are reported beside it."""
    n1 = args.degree + 1
    n2, n3 = n1 * n1, n1 ** 3
    E = conf["elements_per_gpu"]
    dof = E * n3
    peak = peaks.get("hbm_gbs", 6650.0)
    curved = conf.get("geometry") == "curved"
    bf = b_flow(args.degree, curved)
    stage_ms = ms_per_step / 5.0
    ach = value_per_gpu * bf / 1e9
    traffic = None
    prof = sorted(glob.glob(os.path.join(ROOT, "profiles", "*stage_traffic*.json")))
    prof = [p for p in prof if ("curved" in os.path.basename(p)) == curved]
    if prof:
        try:
            traffic = json.load(open(prof[-1])).get("dram_bytes_per_stage")
        except Exception:
            traffic = None
    rl = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
          "kernel": "RK stage = k_gradient + k_update + mortar/pairing kernels (one right-hand side + update)",
          "algorithmic_bytes_per_launch": bf * dof, "bytes_per_dof": bf,
          "per_unit_source": ("SURVEY.md §8(d) B_flow,curved = 400 + 2904/(N+1) B per DOF-update (curved)" if curved
                              else "SURVEY.md §8(d) B_flow = 240 + 2712/(N+1) B per DOF-update (affine)"),
          "mean_launch_ms": stage_ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"}
    extra = {}
    # This implementation's fused dataflow.
    per_kernel = {"update": 8 * E * (20 * n3 + 6 * n2 * 18), "gradient": 8 * E * (5 * n3 + 6 * n2 * 9)}
    if curved:  # + per-node metrics (10 doubles, 13 on the annulus) and per-side face metrics (4 / 6 doubles per
        # face node), read by both kernels
        mw, fw = (13, 6) if args.mesh == "rotor" else (10, 4)
        for k in per_kernel:
            per_kernel[k] += 8 * E * (mw * n3 + 6 * n2 * fw)
    for name, byts in per_kernel.items():
        ms, cnt = kt.get(name, (0.0, 0))
        if cnt:
            t = ms / cnt / 1e3
            extra["k_" + name] = {"mean_launch_ms": t * 1e3, "algorithmic_bytes_per_launch": byts,
                                  "achieved_gbs": byts / t / 1e9, "frac_of_peak": byts / t / 1e9 / peak}
    fused = (per_kernel["update"] + per_kernel["gradient"]) / dof
    extra["fused_dataflow_bytes_per_dof"] = fused
    extra["fused_dataflow_achieved_gbs"] = value_per_gpu * fused / 1e9
    total = sum(v[0] for v in kt.values())
    extra["share_of_step"] = {k: (v[0] / total if total else None) for k, v in kt.items()}
    extra["launches"] = {k: v[1] for k, v in kt.items()}
    return rl, extra


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return

    import torch
    from paper_2008_04356_b200 import capi

    torch.cuda.set_device(local)
    nccl_id = None
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        obj = [capi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    mesh, cfg, conf, dof = workload(args, world)
    s = capi.RankSolver(mesh, cfg, n_ranks=world, rank=rank, device=local, nccl_id=nccl_id)
    s.set_initial_condition(0.0)
    dt = s.suggest_dt(0.5)
    stream = torch.cuda.ExternalStream(s.stream())

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    s.steps_async(dt, args.warmup)
    s.synchronize()
    barrier()
    l0 = s.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        s.steps_async(dt, args.steps)
        ev1.record(stream)
        s.synchronize()
        barrier()
    launches = s.kernel_launches() - l0
    ms = ev0.elapsed_time(ev1)
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = dof * 5 * args.steps / (ms_max / 1e3)

    # Per-kernel timing pass (CUDA events around every launch on the context's stream).
    s.enable_kernel_timing(True)
    s.kernel_timing()
    s.steps_async(dt, 2)
    s.synchronize()
    kt = s.kernel_timing()
    s.enable_kernel_timing(False)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    roof, extra = roofline(kt, conf, args, peaks, value / world, ms_max / args.steps)

    # End-to-end through the C-ABI with pinned host buffers: H2D state, step, D2H state.
    e2e = None
    if not args.no_e2e:
        nbytes = s.size * 8
        h = torch.empty(s.size, dtype=torch.float64).pin_memory()
        hp = h.data_ptr()
        import ctypes
        dp = ctypes.cast(ctypes.c_void_p(hp), ctypes.POINTER(ctypes.c_double))
        s.lib.sdg_get_state(s.h, dp)
        reps = max(2, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            s._check(s.lib.sdg_set_state(s.h, dp))
            s._check(s.lib.sdg_step(s.h, dt))
            s._check(s.lib.sdg_get_state(s.h, dp))
        barrier()
        el = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": dof * 5 * reps / el, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "steps": reps, "path": "sdg_set_state(pinned host) + sdg_step + sdg_get_state(pinned host), wall clock"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": conf.get("scaling", "weak"), "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (analytic initial field)", "config": conf,
                "value_per_gpu": value / world, "dt": dt, "gpu_launches": launches,
                "clocks": clk.summary(), "roofline": roof, "kernels": extra, "e2e": e2e}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args, conf)
        print(json.dumps(line), flush=True)
    s.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
