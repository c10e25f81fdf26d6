"""Benchmark of the B200 sliding-mesh DG right-hand side + RK step.

Default workload: BASELINE.json configs[3], the turbine-scale synthetic the
north star's targets are quoted on -- a 20-degree rotationally periodic annulus
sector, stator / rotor / stator, two sliding interfaces, 1.1M curved hexahedra
(5% warp), N=5 Gauss, fp64, viscous, seeded broadband 1e-2 initial perturbation
(SURVEY §8(d)), strong scaling over the GPUs.  --mesh tgv runs configs[4] (TGV,
affine hexahedra, 64^3 elements per GPU, weak scaling; with --strong its 128^3
strong-scaling mesh, split in y slabs over the GPUs); --mesh warped the same
TGV on curved hexahedra.  configs[0]-[2] are parity cases (tests/).  One "step"
= one 5-stage low-storage RK step (5 right-hand sides + mortars + updates).

metric: BASELINE's "DOF-updates/s (1/PID) per GPU" quantity; `value` is the
whole-job aggregate over all GPUs (E*(N+1)^3 * 5 * steps / time, max over
ranks), `value_per_gpu` = value / n_gpus.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--mesh rotor|tgv|warped]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous).
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
    p.add_argument("--elems", type=int, default=None,
                   help="elements per direction per GPU (weak scaling, default 64); with --strong the whole mesh (default 128)")
    p.add_argument("--strong", action="store_true",
                   help="tgv / warped: configs[4] strong scaling -- --elems is the edge of the WHOLE mesh "
                        "(128 unless given), split in y slabs over the GPUs")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--dry-run", action="store_true", help="stop before the first CUDA call (launcher test)")
    p.add_argument("--mesh", default="rotor", choices=["tgv", "warped", "rotor"],
                   help="tgv: affine hexahedra (configs[4]); warped: the same case on curved hexahedra "
                        "(SDG_MAP_WARP, amplitude 5%% of the element size as in configs[3]); rotor: configs[3], "
                        "1.1M-element stator/rotor/stator 20-degree annulus sector (SDG_MAP_ANNULUS), strong scaling")
    a = p.parse_args()
    if a.elems is None:
        a.elems = 128 if a.strong else 64
    return a


def tgv_mesh(T, elems_x, elems_yz, warp=None, copies=1, yslab=None):
    """Three blocks along x (= BASELINE z); interfaces at 2pi/3, 4pi/3.  Weak scaling over
    `copies` GPUs stacks that many periods of the (2 pi periodic) TGV along the sliding
    direction y and splits it in y slabs through all three blocks (partition 2): every GPU
    holds one identical 64^3 TGV box, both sliding interfaces included."""
    L = 2.0 * math.pi
    base, rem = divmod(elems_x, 3)
    n = [base + (rem == 2), base + (rem == 1), base + (rem == 2)]
    bands = [(n[0], 1.0, 0.0), (n[1], 1.0, 0.2), (n[2], 1.0, 0.0)]
    return T.mesh_spec(bands, ny=elems_yz * copies, nz=elems_yz, width=L, height=L * copies, depth=L, warp=warp,
                       partition=T.PARTITION_YSLAB if (copies > 1 if yslab is None else yslab) else T.PARTITION_LEX), bands


WARP = 0.05  # BASELINE configs[3]: "sinusoidal mesh warping of amplitude 5% of element size"


def rotor_workload(args, world, elements=None, span_div=1):
    """BASELINE configs[3] (turbine-scale synthetic): three axial blocks (stator,
    rotor, stator) of a 20-degree periodic annulus sector r in [0.8, 1] with two
    sliding interfaces, 5% warping inside the blocks (x and r), tip Mach 0.4,
    axial free stream M = 0.3 with the seeded broadband perturbation of SURVEY
    §8(d) (amplitude 1e-2, 8 modes |k| <= 8 in the sector's (x, theta, r),
    mt19937_64(2008043560 + 3)), Re = 8e5 on the mean-radius arc of the sector,
    N = 5.  About 1.1M curved hexahedra (192 axial x 96 around x 60 radial),
    partitioned over the GPUs (strong scaling).  `elements` = (nx, n_theta, n_r)
    and `span_div` (a periodic 1/span_div slice of the sector, same element size)
    shape the CPU sample."""
    from paper_2008_04356_b200 import types as T
    gamma, mach, rho0, u0 = 1.4, 0.3, 1.0, 1.0
    p0 = rho0 * u0 * u0 / (gamma * mach * mach)
    c0 = math.sqrt(gamma * p0 / rho0)
    r_in, r_out = 0.8, 1.0
    omega = 0.4 * c0 / r_out
    sector = math.pi / 9.0
    span = sector / span_div
    chord = 0.5 * (r_in + r_out) * sector
    mu = rho0 * u0 * chord / 8e5
    nx, n_theta, n_r = elements or (192, 96, 60)
    base, rem = divmod(nx, 3)
    n = [base + (rem == 2), base + (rem == 1), base + (rem == 2)]
    bands = [(n[0], 1.0, 0.0), (n[1], 1.0, omega), (n[2], 1.0, 0.0)]
    # Over several GPUs: theta slabs through all three blocks (partition 2), equal work per
    # GPU and rotor/stator mortars mostly rank-local; one GPU: the whole sector.
    mesh = T.annulus_spec(bands, n_theta, n_r, r_in, r_out, length=1.0, warp=WARP, theta_span=span,
                          partition=T.PARTITION_YSLAB if world > 1 else T.PARTITION_LEX)
    case = T.perturbed(T.freestream(rho=rho0, v=(u0, 0.0, 0.0), p=p0), 3, 1e-2, 8, (0.0, 0.0, r_in),
                       (1.0, sector, r_out - r_in), adv=(u0, 0.0, 0.0), cylindrical=True)
    cfg = T.solver_config(args.degree, T.NODES_GAUSS, gamma=gamma, R=1.0, mu=mu, Pr=0.72, case=case)
    n1 = args.degree + 1
    E = nx * n_theta * n_r
    conf = {
        "workload": f"BASELINE configs[3]: stator/rotor/stator annulus sector r in [{r_in}, {r_out}], 20 degrees "
                    f"(rotationally periodic), 2 sliding interfaces, rotor omega {omega:.4f} (tip Mach 0.4), "
                    f"warp {WARP}, axial M=0.3 free stream + seeded broadband 1e-2 density perturbation "
                    f"(8 modes |k|<=8, mt19937_64 seed 2008043563), Re=8e5, "
                    f"{nx}x{n_theta}x{n_r} = {E} curved hexahedra over {world} GPU(s), N={args.degree} Gauss, viscous",
        "mesh": "rotor",
        "geometry": "curved",
        "elements": E,
        "elements_per_gpu": E // world,
        "degree": args.degree,
        "nodes": "gauss",
        "dof": E * n1 ** 3,
        "bands_nx": n,
        "l2_policy": "inputs larger than L2 (state %.0f MB per GPU)" % (E // world * n1 ** 3 * 40 / 1e6),
        "parallelism": (f"dp{world} (theta slabs through all three blocks, NCCL halo + mortar exchange)"
                        if world > 1 else "dp1"),
        "scaling": "strong",
    }
    return mesh, cfg, conf, E * n1 ** 3


def workload(args, world):
    from paper_2008_04356_b200 import types as T
    if args.mesh == "rotor":
        return rotor_workload(args, world)
    curved = args.mesh == "warped"
    strong = bool(getattr(args, "strong", False))
    if strong:  # one mesh of elems^3, y slabs through all three blocks over the GPUs
        mesh, bands = tgv_mesh(T, args.elems, args.elems, warp=WARP if curved else None, copies=1, yslab=world > 1)
    else:
        mesh, bands = tgv_mesh(T, args.elems, args.elems, warp=WARP if curved else None, copies=world)
    cfg = T.solver_config(args.degree, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1.0 / 1600.0, Pr=0.72, case=T.tgv())
    n1 = args.degree + 1
    E = sum(b[0] for b in bands) * args.elems * args.elems * (1 if strong else world)
    geom = (f"curved hexahedra (SDG_MAP_WARP, warp {WARP} of the element size, as BASELINE configs[3]; "
            f"per-node metrics)" if curved else "affine hexahedra")
    conf = {
        "workload": f"BASELINE configs[4]: TGV M=0.1 Re=1600, 3 blocks, 2 planar sliding interfaces (middle +0.2), "
                    + (f"{args.elems}^3 elements over {world} GPU(s) (strong scaling), " if strong
                       else f"{args.elems}^3 elements/GPU, ") + f"N={args.degree} Gauss, viscous, {geom}",
        "mesh": args.mesh,
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
        "scaling": "strong" if strong else "weak",
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


def host_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return ""


def cpu_sample(args, conf):
    """The oracle on the printed workload: the full mesh for the TGV cases (one step
    of 64^3 elements is ~15 s on 16 host threads); for configs[3] a periodic 1/8
    theta slice of the sector -- all 192 axial x 60 radial elements, 12 of the 96
    around, the same element geometry, case and degree (the whole 1.1M-element mesh
    would need ~140 GB of host memory in the oracle).  Per-DOF work is identical, so
    DOF-updates/s compare directly.  Returns (oracle, description)."""
    from oracle import pyoracle as P
    from paper_2008_04356_b200 import types as T
    if args.mesh == "rotor":
        mesh, cfg, sconf, _ = rotor_workload(args, 1, elements=(192, 12, 60), span_div=8)
        desc = f"configs[3] periodic 1/8 theta slice (192x12x60 = {sconf['elements']} elements of the full mesh's geometry)"
    else:
        curved = args.mesh == "warped"
        ne = min(args.elems, 64)  # the 128^3 strong-scaling mesh: a 64^3 TGV box of the same case and degree
        mesh, _ = tgv_mesh(T, ne, ne, warp=WARP if curved else None)
        cfg = T.solver_config(args.degree, T.NODES_GAUSS, gamma=1.4, R=1.0, mu=1.0 / 1600.0, Pr=0.72, case=T.tgv())
        desc = (f"the full printed mesh ({conf['elements_per_gpu']} elements)" if ne == args.elems
                else f"a {ne}^3-element TGV box of the printed case (the printed mesh has {conf['elements']} elements)")
    o = P.Oracle3D(mesh, cfg)
    o.set_initial_condition(0.0)
    return o, desc


def time_oracle(o, args, max_steps, budget_s, warmup=1):
    dt = 0.25 * o.suggest_dt(0.5)
    for _ in range(warmup):
        o.step(dt, 1)
    steps, t0 = 0, time.perf_counter()
    while steps < max_steps and (steps == 0 or time.perf_counter() - t0 < budget_s):
        o.step(dt, 1)
        steps += 1
    return steps, time.perf_counter() - t0


def cpu_baseline(args, conf, budget_s=20.0, max_steps=100, warmup=1):
    """The 3D CPU oracle (restatement of the reference path, 'port'; the reference
    library itself is 2D) with all host threads on the printed workload
    (cpu_sample), timed over whole RK steps after `warmup` steps."""
    from oracle import pyoracle as P
    threads = os.cpu_count() or 1
    P.oracle_lib().orc_set_threads(threads)
    t_setup = time.perf_counter()
    o, desc = cpu_sample(args, conf)
    setup = time.perf_counter() - t_setup
    steps, el = time_oracle(o, args, max_steps, budget_s, warmup)
    dof = o.n_elements * (args.degree + 1) ** 3
    out = {"value": dof * 5 * steps / el, "unit": UNIT, "cores": threads, "kind": "port",
           "steps_timed": steps, "ms_per_step_of_sample": 1e3 * el / steps, "sample_dof": dof,
           "sample": f"oracle/sdg3d.cpp (OpenMP, {threads} threads, {host_model()}) on {desc}, N={args.degree}, "
                     f"{dof} DOF: {steps} RK step(s) in {el:.1f} s after {warmup} warm-up step(s) "
                     f"(setup {setup:.0f} s untimed)"}
    try:
        out["reference_2d"] = reference_2d(args.degree, seconds=8.0)
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
    """--impl reference: the CPU implementation of the path on the host cores, on
    this arm's workload (cpu_sample).  The reference library itself is 2D-only
    (SURVEY §0), so the 3D restatement of its algorithm (oracle/sdg3d.cpp, 'port')
    runs this arm.  Steps are whole RK steps of the sample; K and W are capped so
    the run stays within a few minutes."""
    if rank != 0:
        return
    mesh, cfg, conf, dof = workload(args, world)
    base = cpu_baseline(args, conf, budget_s=60.0, max_steps=args.steps, warmup=min(args.warmup, 1))
    line = {"metric": METRIC, "value": base["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": base["ms_per_step_of_sample"], "higher_is_better": True,
            "scaling": conf.get("scaling", "weak"),
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded analytic initial field)",
            "config": conf, "impl": "reference", "cpu_baseline": base,
            "ms_per_step_note": "one RK step of the bounded sample (cpu_baseline.sample), not of the whole workload",
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
    # ncu DRAM bytes of the stage's element kernels, from a capture of this exact
    # workload (tools/summarize_ncu.py writes the workload key into the file).
    traffic, traffic_src, flops_per_dof = None, None, None
    key = {"mesh": conf.get("mesh"), "degree": args.degree, "elements_per_gpu": E}
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_stage_traffic.json"))):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        if d.get("workload") == key:
            traffic, traffic_src = d.get("dram_bytes_per_stage"), os.path.relpath(p, ROOT)
            flops_per_dof = d.get("fp64_flops_per_dof")
    rl = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
          "kernel": "RK stage = k_gradient + k_update + mortar/pairing kernels (one right-hand side + update)",
          "algorithmic_bytes_per_launch": bf * dof, "bytes_per_dof": bf,
          "per_unit_source": ("SURVEY.md §8(d) B_flow,curved = 400 + 2904/(N+1) B per DOF-update (curved)" if curved
                              else "SURVEY.md §8(d) B_flow = 240 + 2712/(N+1) B per DOF-update (affine)"),
          "mean_launch_ms": stage_ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)",
          "traffic_source": traffic_src}
    # The FP64 side of the roofline (north star: "fraction of the HBM/FP64 roofline"): FP64 flops per
    # DOF-update counted by ncu on this workload (same capture as `traffic`), against the DFMA peak
    # measured by tools/fp64_peak.cu on this pool's B200 (profiles/*_fp64_peak.json).
    fp64_peak, fp64_src = None, None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_fp64_peak.json"))):
        try:
            fp64_peak, fp64_src = json.load(open(p))["fp64_dfma_tflops"], os.path.relpath(p, ROOT)
        except Exception:
            pass
    if flops_per_dof and fp64_peak:
        tf = value_per_gpu * flops_per_dof / 1e12
        rl["fp64"] = {"achieved": tf, "peak": fp64_peak, "unit": "TFLOP/s", "frac": tf / fp64_peak,
                      "flops_per_dof": flops_per_dof, "flops_source": traffic_src, "peak_source": fp64_src,
                      "intensity_flop_per_byte": (flops_per_dof * dof / traffic) if traffic else None}
    extra = {}
    # This implementation's fused dataflow, doubles per element.
    #   affine: k_gradient_ws reads U, own + neighbour traces, writes Fv.n; k_update_bulk reads U, the RK
    #   register, own + neighbour traces and Fv.n, writes U, register, traces.
    #   curved (even N+1): k_gradient_cv also reads Ja, 1/J (10 rows) and 4 face-metric rows and writes the
    #   node's stress / heat flux (9); k_update_cv reads those 9, all node-metric rows and the face-metric rows
    #   it uses instead of evaluating the gradient again.
    #   per face node: own trace 5 + own Fv.n 4 + neighbour trace 5 + Fv.n 4 read, new trace 5 written (update);
    #   own + neighbour trace read, Fv.n written (gradient).
    per_kernel = {"update": 8 * E * (20 * n3 + 6 * n2 * 23), "gradient": 8 * E * (5 * n3 + 6 * n2 * 14)}
    even = n1 % 2 == 0
    if even:  # the node's stress / heat flux (9 doubles) handed from the gradient to the update kernel
        per_kernel["gradient"] += 8 * E * 9 * n3
        per_kernel["update"] += 8 * E * 9 * n3
    if curved:
        mw, fw_u = (13, 5) if args.mesh == "rotor" else (10, 4)
        if even:
            per_kernel["gradient"] += 8 * E * (10 * n3 + 6 * n2 * 4)
            per_kernel["update"] += 8 * E * (mw * n3 + 6 * n2 * fw_u)
        else:  # plain-load kernels: every metric row in both, gradient evaluated twice
            for k in per_kernel:
                per_kernel[k] += 8 * E * (mw * n3 + 6 * n2 * (6 if args.mesh == "rotor" else 4))
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


def relaunch(args):
    """`--gpus N` outside torchrun: N ranks through torch.distributed.run (the
    driver's own launch line), one per GPU."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return

    import torch
    from paper_2008_04356_b200 import capi

    nccl_id = None
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        obj = [capi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    mesh, cfg, conf, dof = workload(args, world)
    if args.dry_run:
        # Everything up to the first CUDA call: the rank's share of the partition.
        plan = capi.plan(mesh, world, rank)
        print(json.dumps({"rank": rank, "world": world, "local_rank": local, "nccl_id_bytes": len(nccl_id or b""),
                          "elements": len(plan["elements"]), "interior_run": plan["interior_run"],
                          "halo_peers": [h["partner"] for h in plan["halo"]], "config": conf}), flush=True)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    torch.cuda.set_device(local)
    s = capi.RankSolver(mesh, cfg, n_ranks=world, rank=rank, device=local, nccl_id=nccl_id)
    s.set_initial_condition(0.0)
    # CFL 0.5 as BASELINE configs[0]; N >= 6 runs at 0.25: at 0.5 the scheme itself (oracle and device alike) is
    # unstable on the TGV at N = 7 and leaves the admissible set after ~20 steps.  Throughput does not depend on dt.
    cfl = 0.5 if args.degree <= 5 else 0.25
    dt = s.suggest_dt(cfl)
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
                "data": "synthetic (seeded analytic initial field; no dataset)", "config": conf,
                "metric_note": "value = whole-job aggregate over n_gpus; value_per_gpu = value / n_gpus",
                "value_per_gpu": value / world, "dt": dt, "cfl": cfl, "gpu_launches": launches,
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
