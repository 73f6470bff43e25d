"""Benchmark: 4D Vlasov DOF-updates/s per Strang step on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
                    [--impl vpb|reference] [--no-e2e] [--no-cpu-baseline]
                    [--per-step | --graph]

One "step" is one Strang step of the reference's ``strang_step`` (six
sweeps, density, field solve, v-shift tables, the non-finite checks).  The
timed K steps run through ``advance(field, tau, K)``, the public multi-step
API (the reference's ``run`` loop without diagnostics): adjacent x half steps
of consecutive steps share one HBM pass ("fast" arithmetic: composed
three-cell stencils, equal to the separate sweeps up to round-off; with
VPB_ARITH=exact bitwise the K ``strang_step`` calls).  K defaults to the
configuration's BASELINE step count (config 2: 100 steps).  ``per_call`` in the JSON line times K separate
``strang_step(consume=True)`` calls (what the reference's ``bench_step``
times, /root/reference/pkg/src/slvp/bench.py:54-68); ``--per-step`` makes
that the headline.  The default workload is BASELINE config 2 (Landau 4D,
64^4 cells, degree 2 = 192^4 = 1.36e9 dofs, 10.9 GB per copy of f, dt =
0.05), the configuration the metric is quoted on that fits one GPU.

Timing: W untimed warm-up steps, then exactly K steps bracketed by a
barrier + torch.cuda.synchronize(), timed with CUDA events on the launching
stream; max over ranks.  The field (10.9 GB) is ~87x the 126 MB L2, so no
explicit L2 flush is needed.  SM clocks / throttle reasons are sampled with
nvidia-smi during the timed region.

``e2e``: Strang steps of a field resident in pinned HOST memory through the
public ``host_steps(HostField, tau, K)`` (what a reference user holding f on
the host sees): every step copies f host->device and back, pipelined per v2
block against the plane-local x passes, with the D2H of step m and the H2D
of step m+1 running concurrently (paper_1803_02143_b200/hoststep.py).

``roofline``: the dominant kernel (most device time per step) measured by
CUDA events around its launches in the timed steps; algorithmic bytes = 16
B per dof per sweep (one fp64 read + one write).

``cpu_baseline`` / ``--impl reference``: the UNMODIFIED reference package
(pip-installed into oracle/_ref/site by oracle/build.py) through its own
public API: ``slvp.strang_step(consume=True)`` on every host thread, full
steps of the same configuration under its bench_step protocol
(oracle/refstep.py); cpu_baseline = one warm-up + one timed step, the
reference arm = one warm-up + as many steps as fit in --ref-budget.  Only a
configuration that does not fit host RAM falls back to the scaled slab
sample (oracle/refarm.py), labelled EXTRAPOLATED.

Multi-GPU (torchrun, N > 1): the dG field is sharded along x1 (x1 x x2 on
8 GPUs when the merged pass's halo does not fit an x1 shard) with NCCL halo
exchange and a rho all-gather (paper_1803_02143_b200.dist,
ShardedSolver.advance); the global grid is fixed (``scaling: strong``).  ``--replicas`` runs N independent full-size replicas instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "4D Vlasov DOF-updates/s per Strang step at 1/2/4/8 B200; % of HBM roofline"
UNIT = "DOF-updates/s"

CONFIGS = {
    # BASELINE.json configs (degree 2 == dg_order 3)
    "cfg1": dict(problem="landau4d", method="dg", dofs=48, order=3, tau=0.1, nsteps=20,
                 label="BASELINE config 1: Landau 4D, 16^4 cells, degree 2 (48^4 dofs), dt=0.1"),
    "cfg2": dict(problem="landau4d", method="dg", dofs=192, order=3, tau=0.05, nsteps=100,
                 label="BASELINE config 2: Landau 4D, 64^4 cells, degree 2 (192^4 = 1.36e9 dofs), dt=0.05"),
    "cfg3": dict(problem="twostream4d_baseline", method="dg", dofs=128, order=2, tau=0.1, nsteps=200,
                 label="BASELINE config 3: two-stream 4D, 64^4 cells, degree 1 (128^4 dofs), dt=0.1"),
    "cfg4": dict(problem="landau4d", method="spline", dofs=128, order=0, tau=0.1, nsteps=50,
                 label="BASELINE config 4: Landau 4D cubic spline, 128^4 points, dt=0.1"),
    "cfg5": dict(problem="landau4d", method="dg", dofs=288, order=3, tau=0.05, nsteps=20,
                 label="BASELINE config 5: Landau 4D, 96^4 cells, degree 2 (288^4 = 6.9e9 dofs), dt=0.05"),
}

BYTES_PER_DOF_SWEEP = 16  # read + write one fp64 per dof
L2_BYTES = 126 * 2**20


def sweeps_per_launch(label: str) -> int:
    """1-D sweeps one launch of a kernel group performs (labels of driver.enqueue_steps)."""
    name = label[len("sweep_"):].replace("_rho", "")
    return {"x12": 2, "v12": 2, "x12x12": 4, "x1x2": 2, "x2x2": 2, "xx2": 2}.get(name, 1)


def fp64_peak_gops() -> float:
    """fp64 vector issue peak of the device: SMs x 64 lanes x max SM clock."""
    try:
        import torch

        props = torch.cuda.get_device_properties(torch.cuda.current_device())
        sms = props.multi_processor_count
    except Exception:  # noqa: BLE001
        sms = 148
    mhz = 1965.0
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        mhz = float(json.loads(p.read_text()).get("sm_max_mhz", mhz))
    return sms * 64 * mhz * 1e6 / 1e9


def l2_note(copy_bytes: int) -> str:
    if copy_bytes > 8 * L2_BYTES:
        return f"inputs ({copy_bytes / 1e9:.3g} GB per copy of f) >> 126 MB L2; no flush"
    return (f"inputs ({copy_bytes / 1e6:.3g} MB per copy of f) fit in L2: warm-L2 timing of a "
            "launch-bound configuration, not a headline number")


def group_times(ev: list, labels: list) -> dict:
    """label -> [total ms, count] from consecutive CUDA events (a label runs
    until the next event)."""
    groups: dict = {}
    for i in range(len(ev) - 1):
        if labels[i] is None:
            continue
        dt = ev[i].elapsed_time(ev[i + 1])
        g = groups.setdefault(labels[i], [0.0, 0])
        g[0] += dt
        g[1] += 1
    return groups


def load_traffic(cfg_name: str, label: str):
    """ncu DRAM bytes (read + write) per launch of the kernel behind ``label``
    on this workload, from the committed capture summary profiles/traffic.json
    (null when that kernel has not been captured)."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    ent = json.loads(p.read_text()).get(cfg_name, {}).get(label)
    if not ent or ent.get("arithmetic") not in (None, os.environ.get("VPB_ARITH", "fast")):
        return None
    return float(ent["dram_bytes_per_launch"])


def load_peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampling
# ---------------------------------------------------------------------------
REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons.  Started before
    the warm-up (the tool takes a while to come up); only samples whose
    timestamps fall inside [begin, end] of the timed region are summarised."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"vpb_clocks_{os.getpid()}.csv"
        self.t0 = self.t1 = None

    def start(self):
        q = ("timestamp,clocks.sm,clocks.max.sm,"
             + ",".join(f"clocks_event_reasons.{r}" for r in REASONS))
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
            return self
        deadline = time.time() + 10.0
        while time.time() < deadline and self.path.stat().st_size == 0:
            time.sleep(0.05)
        return self

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()
        time.sleep(0.12)  # let the last in-window sample land

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def __enter__(self):
        return self.start()

    def __exit__(self, *exc):
        self.stop()

    def summary(self) -> dict | None:
        if self.proc is None or not self.path.exists():
            return None
        from datetime import datetime

        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 3 + len(REASONS):
                continue
            try:
                ts = datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        try:
            self.path.unlink()
        except OSError:
            pass
        if not rows:
            return None
        inside = [r for r in rows if self.t0 is not None and self.t0 <= r[0] <= (self.t1 or r[0])]
        use = inside or sorted(rows, key=lambda r: abs(r[0] - (self.t0 or r[0])))[:3]
        active = set()
        for r in use:
            for name, v in zip(REASONS, r[3]):
                if v.lower().startswith("active"):
                    active.add(name)
        return {"sm_mhz": float(np.median([r[1] for r in use])),
                "sm_max_mhz": float(max(r[2] for r in use)), "reasons": sorted(active),
                "samples": len(use), "in_window": bool(inside)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
# The JSON line goes to the process's original stdout; everything else that
# writes to file descriptor 1 (NCCL's version banner, library chatter) is
# sent to stderr, so stdout carries exactly one JSON line.
_JSON_OUT = None


def protect_stdout() -> None:
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit_line(line: dict) -> None:
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def maybe_init(world: int, local: int, backend: str, force: bool = False):
    """Process group for N > 1 (torchrun); ``force`` also creates it for a
    single rank (``--sharded``: the multi-GPU code path, NCCL included, on a
    one-GPU box)."""
    import torch
    import torch.distributed as dist

    if (world > 1 or force) and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", str(world))
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return dist if (world > 1 or force) else None


def barrier(d, device=None):
    if d is not None:
        if device is not None:
            d.barrier(device_ids=[device])
        else:
            d.barrier()


def allreduce_max(d, value: float) -> float:
    if d is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    d.all_reduce(t, op=d.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def _host_ram_bytes() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_reference(cfg: dict, *, warmup: int = 1, max_steps: int = 1,
                  budget_s: float = 240.0, threads: int | None = None) -> dict:
    """The unmodified reference ``slvp.strang_step`` (oracle/_ref/site) timed
    on full steps of the configuration on this box's host cores
    (oracle/refstep.py).  A configuration whose reference run does not fit
    host RAM (2 copies of f above 80 % of MemAvailable) falls back to the scaled
    slab sample of the reference's compiled kernels (oracle/refarm.py) and
    says so in ``sample``."""
    need = 2 * 8 * int(cfg["dofs"]) ** 4  # strided dG steps in place (RSS ~1 copy at cfg2)
    avail = _host_ram_bytes()
    from oracle import build

    if build.load_ref_pkg() is not None and (avail == 0 or need < 0.8 * avail):
        from oracle import refstep

        return refstep.time_steps(cfg["problem"], cfg["method"], cfg["dofs"], cfg["order"],
                                  cfg["tau"], threads=threads, warmup=warmup,
                                  max_steps=max_steps, budget_s=budget_s)
    from oracle import refarm

    r = refarm.reference_step_rate(cfg["problem"], cfg["method"], cfg["dofs"], cfg["order"],
                                   cfg["tau"], threads=threads)
    r["sample"] = ("EXTRAPOLATED (full-size reference run needs %.0f GB, host has %.0f GB "
                   "available): " % (need / 1e9, avail / 1e9)) + r["sample"]
    r["steps_timed"] = 0
    return r


def run_reference_arm(args, cfg_name: str, cfg: dict) -> None:
    """``--impl reference``: the reference's own strang_step on every host
    thread, full steps of the same configuration (bench_step protocol), as
    many as fit in ``--ref-budget`` seconds (at most ``--steps``), after one
    warm-up step.  Plus a 1-core figure (config 1, full steps)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    r = cpu_reference(cfg, warmup=1, max_steps=args.steps, budget_s=args.ref_budget)
    one = cpu_reference(CONFIGS["cfg1"], warmup=1, max_steps=3, budget_s=30.0, threads=1)
    value = r["dof_per_s"]
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": int(r.get("steps_timed", 0)), "warmup": int(r.get("warmup", 0)),
        "requested": {"steps": args.steps, "warmup": args.warmup,
                      "note": "full reference steps take tens of seconds: one warm-up step, "
                              "then as many timed steps as fit in --ref-budget"},
        "ms_per_step": r["step_s"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE initial condition, no dataset)",
        "config": {"workload": cfg_name, "description": cfg["label"],
                   "dofs": int(cfg["dofs"]) ** 4, "parallelism": "cpu-threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["threads"],
                         "kind": r["kind"], "sample": r["sample"]},
        "samples_s": r.get("samples_s"),
        "one_core": {"value": one["dof_per_s"], "unit": UNIT, "cores": 1,
                     "config": "cfg1", "ms_per_step": one["step_s"] * 1e3,
                     "sample": one["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host_threads": r["threads"],
    }
    emit_line(line)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_sharded(args, cfg_name: str, cfg: dict, d, world: int, rank: int, local: int) -> None:
    """N > 1: one shard of the field per GPU (x1, or x1 x x2 at 8 GPUs), NCCL
    halo exchange + rho all-gather (paper_1803_02143_b200.dist); strong
    scaling (the global grid is fixed)."""
    import torch

    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200 import dist

    problem = vpb.problem_spec(cfg["problem"])
    grid = vpb.make_grid(problem, cfg["method"], cfg["dofs"], dg_order=cfg["order"])
    N = grid.total_dof
    tau = cfg["tau"]
    if cfg["method"] == "dg" and args.layout == "v":
        # velocity sharding (the paper's decomposition): v2 slabs, local x
        # passes, one v2 halo exchange per step (dist.VShardedSolver)
        solver = dist.VShardedSolver(grid, dist.TorchComm(), [rank], world,
                                     peer_halos=args.peer_halos)
        local_f = lambda: solver.local(solver.f[rank], rank)  # noqa: E731
        layout = (f"v2-shard x{world} (local x passes; v2 halos of {solver.H} cells per side "
                  + ("read in place from the neighbours' buffers over NVLink (CUDA IPC)"
                     if args.peer_halos else "by zero-copy NCCL send/recv")
                  + "; rho partials all-gathered)")
    elif cfg["method"] == "dg":
        # the process grid (x1 x x2: 4 x 2 at 8 GPUs, emulated 2.56 ms per rank
        # at config 2 vs 4.37 for 8 x1 shards) when its merged stencil passes
        # apply, else x1 shards, else the process grid with per-sweep halos
        p1, p2 = dist.process_grid(world)
        solver = None
        for a, b in ((p1, p2), (world, 1)):
            cand = dist.ShardedSolver(grid, dist.Decomposition(grid, a, b), dist.TorchComm(),
                                      [rank])
            if cand._stencil_ready(tau) and cand._merged_halo_fits(tau):
                solver, p1, p2 = cand, a, b
                break
        if solver is None:
            solver = dist.ShardedSolver(grid, dist.Decomposition(grid, p1, p2),
                                        dist.TorchComm(), [rank])
        local_f = lambda: solver.shards[rank].f  # noqa: E731
        layout = (f"x-shard {p1}x{p2} (NCCL halos + rho allgather"
                  + ("; merged x passes as halo-exchanged stencil passes)"
                     if solver._stencil_ready(tau) else ")"))
    else:
        solver = dist.SplineShardedSolver(grid, dist.TorchComm(), [rank], world)
        local_f = lambda: solver.a[rank][0]  # noqa: E731
        layout = f"v2-shard x{world} <-> x2-shard (2 NCCL all-to-alls per step, rho allreduce)"
    solver.initialize(problem)
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local).start()

    labels: list = []
    ev: list = []

    def mark(label):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        ev.append(e)
        labels.append(label)

    def steps(k: int, timer=None) -> None:
        # dG: advance() merges the x half steps of consecutive steps into one
        # halo-exchanged stencil pass per step (x1-sharded layouts)
        if hasattr(solver, "advance"):
            solver.advance(tau, k, timer=timer)
        else:
            for _ in range(k):
                solver.step(tau)

    steps(args.warmup)
    from paper_1803_02143_b200 import _lib

    barrier(d, local)
    torch.cuda.synchronize()
    n_launch0 = _lib.load().vpb_launch_count()
    solver._halo_bytes = 0
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    clocks.begin()
    start.record(stream)
    steps(args.steps, timer=mark if hasattr(solver, "advance") else None)
    end.record(stream)
    torch.cuda.synchronize()
    clocks.end()
    clocks.stop()
    gpu_launches = _lib.load().vpb_launch_count() - n_launch0  # rank 0's kernels
    halo_bytes = getattr(solver, "_halo_bytes", 0) / max(1, args.steps)
    barrier(d, local)
    total_ms = allreduce_max(d, start.elapsed_time(end))
    ms_per_step = total_ms / args.steps
    value = N * args.steps / (total_ms * 1e-3)
    # per-group device time on this rank; the dominant sweep kernel on the
    # same basis as the 1-GPU line: 16 B per LOCAL dof per launch
    groups = group_times(ev, labels)
    n_local = local_f().numel()
    per_kernel = {k: {"avg_ms": v[0] / v[1], "launch_groups": v[1],
                      "share_of_step": v[0] / total_ms} for k, v in sorted(groups.items())}
    sweeps = {k: v for k, v in groups.items() if k.startswith("sweep_")}
    peak, peak_kind = load_peaks()
    dom = max(sweeps, key=lambda k: sweeps[k][0]) if sweeps else None
    for k in sweeps:
        t = per_kernel[k]["avg_ms"] * 1e-3
        per_kernel[k]["achieved_gbs"] = BYTES_PER_DOF_SWEEP * n_local / t / 1e9
        per_kernel[k]["frac"] = per_kernel[k]["achieved_gbs"] / peak
        per_kernel[k]["sweeps_per_launch"] = sweeps_per_launch(k)
    dom_frac = allreduce_max(d, per_kernel[dom]["frac"]) if dom else None
    # e2e: each rank's slab from pinned host memory, step, back to the host
    e2e = None
    if not args.no_e2e:
        host = torch.empty(local_f().numel(), dtype=torch.float64, pin_memory=True)
        host.copy_(local_f())
        k_e2e = max(1, min(args.steps, args.e2e_steps))
        barrier(d, local)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(k_e2e):
            local_f().copy_(host, non_blocking=True)
            if hasattr(solver, "advance"):
                solver.advance(tau, 1)
            else:
                solver.step(tau)
            host.copy_(local_f(), non_blocking=True)
        s1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = allreduce_max(d, s0.elapsed_time(s1))
        nbytes = 8 * host.numel()
        e2e = {"value": N * k_e2e / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": nbytes * world, "d2h_bytes_per_step": nbytes * world,
               "steps": k_e2e, "ms_per_step": e2e_ms / k_e2e,
               "path": "per-rank pinned host slab -> H2D -> sharded step -> D2H"}
    step_gbs_local = 6 * BYTES_PER_DOF_SWEEP * n_local / (ms_per_step * 1e-3) / 1e9
    if rank == 0:
        emit_line({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE initial condition on the named grid; no dataset)",
            "config": {"workload": cfg_name, "description": cfg["label"], "dofs": N,
                       "parallelism": layout,
                       "l2": l2_note(8 * N // world)},
            "roofline": {"bound": "hbm",
                         "achieved": (per_kernel[dom]["achieved_gbs"] if dom else None),
                         "peak": peak, "unit": "GB/s", "frac": per_kernel[dom]["frac"] if dom
                         else None, "frac_max_over_ranks": dom_frac,
                         "traffic": None, "kernel": dom,
                         "algorithmic_bytes_per_launch": BYTES_PER_DOF_SWEEP * n_local,
                         "basis": "rank 0's dominant sweep kernel, 16 B per local dof per "
                                  "launch / average launch time (same basis as the 1-GPU line)",
                         "step_frac": step_gbs_local / peak,
                         "step_bytes": 6 * BYTES_PER_DOF_SWEEP * n_local,
                         "peak_source": peak_kind},
            "kernels": per_kernel,
            "comm_bytes_per_step": {"halo_send": halo_bytes,
                                    "rho_allgather": 8 * (grid.dims4[0] // max(1, cfg["order"]))
                                    * (grid.dims4[1] // max(1, cfg["order"]))
                                    if cfg["method"] == "dg" else None},
            "e2e": e2e, "cpu_baseline": None, "clocks": clocks.summary(),
            "gpu_launches": int(gpu_launches),
        })
    if d is not None:
        d.destroy_process_group()


def run_vpb(args, cfg_name: str, cfg: dict) -> None:
    import torch

    world, rank, local = dist_env()
    d = maybe_init(world, local, "nccl", force=args.sharded)
    torch.cuda.set_device(local)
    if (world > 1 or args.sharded) and not args.replicas:
        return run_sharded(args, cfg_name, cfg, d, world, rank, local)
    import paper_1803_02143_b200 as vpb
    from paper_1803_02143_b200 import driver

    problem = vpb.problem_spec(cfg["problem"])
    grid = vpb.make_grid(problem, cfg["method"], cfg["dofs"], dg_order=cfg["order"])
    N = grid.total_dof
    tau = cfg["tau"]
    field = vpb.initialize(problem, grid)
    st = driver.step_state(grid)
    stream = torch.cuda.current_stream()

    clocks = ClockSampler(local).start()
    from paper_1803_02143_b200 import _lib

    lib = _lib.load()
    mode = (("graph" if args.per_step else "advance-graph") if args.graph
            else ("per-step" if args.per_step else "merged"))
    dev = torch.device("cuda", local)
    nslot = st.flags.numel()

    def flags_for(k):
        return (torch.zeros((k, nslot), dtype=torch.int32, device=dev),
                torch.zeros((k, st.stats.numel()), dtype=torch.float64, device=dev))

    def run_steps(k, timer=None, how=None):
        """k steps through the public step API of the selected mode."""
        how = how or mode
        if how == "merged":  # == driver.advance(field, tau, k, consume=True)
            fl, sts = flags_for(k)
            driver.enqueue_steps(field, tau, k, st, fl, sts, timer)
            driver.check_steps(st, fl, sts, None, tau)
        else:  # == k x strang_step(field, tau, consume=True)
            for _ in range(k):
                driver.enqueue_step(field, tau, st, timer=timer)
                driver.check_step(st, None)

    run_steps(args.warmup, how="merged" if mode in ("merged", "advance-graph") else "per-step")

    # --- timed region: K steps, events per kernel group
    labels: list = []
    ev: list = []

    def mark(label):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        ev.append(e)
        labels.append(label)

    graph = None
    n_launch0 = lib.vpb_launch_count()
    if mode in ("graph", "advance-graph"):
        # the per-kernel breakdown comes from an eager pass of K steps; the
        # headline timing replays the steps from CUDA graphs (per step, or the
        # whole K-step advance() block)
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_steps(args.steps, timer=mark, how="per-step" if mode == "graph" else "merged")
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(stream)
        torch.cuda.synchronize()
        eager_ms = e0.elapsed_time(e1)
        eager_launches = lib.vpb_launch_count() - n_launch0
        if mode == "graph":
            graph = driver.StepGraph(field, tau)
            for _ in range(args.warmup):
                graph.step()
        else:
            graph = driver.AdvanceGraph(field, tau, args.steps)
            graph.advance()
    barrier(d, local)
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    clocks.begin()
    start.record(stream)
    if mode == "advance-graph":
        graph.advance()
    elif graph is not None:
        for _ in range(args.steps):
            graph.step()
    else:
        run_steps(args.steps, timer=mark)
    end.record(stream)
    torch.cuda.synchronize()
    clocks.end()
    clocks.stop()
    # kernels launched through libvpb200 in the timed steps (graph replays
    # launch the same kernels the eager pass counted)
    gpu_launches = eager_launches if graph is not None else lib.vpb_launch_count() - n_launch0
    barrier(d, local)
    total_ms = start.elapsed_time(end)
    total_ms = allreduce_max(d, total_ms)
    ms_per_step = total_ms / args.steps
    value = world * N * args.steps / (total_ms * 1e-3)
    breakdown_ms = eager_ms if graph is not None else total_ms

    # the per-call API (one strang_step per step) for comparison
    per_call = None
    if mode != "per-step":
        barrier(d, local)
        torch.cuda.synchronize()
        p0 = torch.cuda.Event(enable_timing=True)
        p1 = torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        run_steps(args.steps, how="per-step")
        p1.record(stream)
        torch.cuda.synchronize()
        pc_ms = allreduce_max(d, p0.elapsed_time(p1))
        per_call = {"api": "strang_step(consume=True) per step", "ms_per_step": pc_ms / args.steps,
                    "value": world * N * args.steps / (pc_ms * 1e-3), "unit": UNIT}

    # per-group device time
    groups = group_times(ev, labels)
    sweeps = {k: v for k, v in groups.items() if k.startswith("sweep_")}
    dom = max(sweeps, key=lambda k: sweeps[k][0])
    dom_avg_ms = sweeps[dom][0] / sweeps[dom][1]
    peak, peak_kind = load_peaks()
    achieved = BYTES_PER_DOF_SWEEP * N / (dom_avg_ms * 1e-3) / 1e9
    step_gbs = 6 * BYTES_PER_DOF_SWEEP * N / (ms_per_step * 1e-3) / 1e9
    per_kernel = {k: {"avg_ms": v[0] / v[1], "launch_groups": v[1],
                      "share_of_step": v[0] / breakdown_ms}
                  for k, v in sorted(groups.items())}
    # 1-D sweeps done per launch (fused passes chain several in registers);
    # dG sweeps cost 4P-1 fp64 operations per dof, without contraction
    fp64_peak = fp64_peak_gops()
    for k, v in per_kernel.items():
        if k.startswith("sweep_"):
            t = v["avg_ms"] * 1e-3
            nsw = sweeps_per_launch(k)
            v["achieved_gbs"] = BYTES_PER_DOF_SWEEP * N / t / 1e9
            v["frac"] = v["achieved_gbs"] / peak
            v["sweeps_per_launch"] = nsw
            v["unfused_equivalent_frac"] = nsw * v["frac"]
            if cfg["method"] == "dg":
                ops = nsw * (4 * cfg["order"] - 1)
                if k.startswith("sweep_x12x12") and vpb.arithmetic() == "fast":
                    ops = 2 * 3 * cfg["order"]  # two composed 3-cell stencils (FMA)
                v["fp64_gops"] = ops * N / t / 1e9
                v["fp64_frac"] = v["fp64_gops"] / fp64_peak

    # --- e2e through the public API with host-resident f
    e2e = None
    if not args.no_e2e:
        from paper_1803_02143_b200 import hoststep

        host = hoststep.HostField.from_field(field)
        field = graph = None  # the device-resident field is done: free its copy (config 5)
        torch.cuda.empty_cache()
        k_e2e = max(1, min(args.steps, args.e2e_steps))
        hoststep.host_steps(host, tau, 1, blocks=args.e2e_blocks)  # warm-up (buffers, tables)
        barrier(d, local)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        w0 = time.perf_counter()
        # check_steps inside host_steps synchronises after the last D2H, so the
        # end event is recorded on the compute stream after every copy completed
        hoststep.host_steps(host, tau, k_e2e, blocks=args.e2e_blocks)
        s1.record(stream)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - w0) * 1e3
        e2e_ms = allreduce_max(d, s0.elapsed_time(s1))
        e2e = {"value": world * N * k_e2e / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N, "steps": k_e2e,
               "ms_per_step": e2e_ms / k_e2e, "wall_ms_per_step": wall_ms / k_e2e,
               "pcie_gbs_per_direction": 8 * N / (e2e_ms / k_e2e * 1e-3) / 1e9,
               "blocks": args.e2e_blocks,
               "path": "host_steps(HostField): f in pinned host memory between steps; per "
                       "step every v2 block goes H2D -> opening x pass, whole-field density/"
                       "field solve/v pass, closing x pass -> D2H; H2D of step m+1 overlaps "
                       "D2H of step m block by block (hoststep.py)"}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference(cfg, warmup=1, max_steps=1)
        cpu = {"value": r["dof_per_s"], "unit": UNIT, "cores": r["threads"], "kind": r["kind"],
               "sample": r["sample"]}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE initial condition on the named grid; no dataset)",
            "config": {"workload": cfg_name, "description": cfg["label"], "dofs": N,
                       "bytes_per_copy": 8 * N, "l2": l2_note(8 * N),
                       "parallelism": "replicas" if world > 1 else "single-gpu"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": (args.traffic if args.traffic is not None
                                     else load_traffic(cfg_name, dom)),
                         "kernel": dom,
                         "peak_source": peak_kind,
                         "algorithmic_bytes_per_launch": BYTES_PER_DOF_SWEEP * N,
                         "step_frac": step_gbs / peak,
                         "step_bytes": 6 * BYTES_PER_DOF_SWEEP * N,
                         "sweeps_per_launch": per_kernel[dom]["sweeps_per_launch"],
                         "unfused_equivalent_frac": per_kernel[dom]["unfused_equivalent_frac"],
                         "fp64_frac": per_kernel[dom].get("fp64_frac"),
                         "fp64_peak_gops": fp64_peak if cfg["method"] == "dg" else None,
                         "fp64_peak_source": "derived: SMs x 64 fp64 lanes x max SM clock "
                                             "(not measured)"},
            "kernels": per_kernel,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gpu_launches": int(gpu_launches),
            "cuda_graph": bool(args.graph),
            "arithmetic": vpb.arithmetic(),
            "step_api": {"merged": "advance(field, tau, K): K Strang steps, adjacent x half "
                                   "steps share one HBM pass ('fast': composed 3-cell "
                                   "stencils; 'exact': the four sweeps bitwise)",
                         "per-step": "strang_step(consume=True) per step",
                         "graph": "strang_step per step replayed from CUDA graphs",
                         "advance-graph": "advance(field, tau, K) replayed from a CUDA graph "
                                          "(driver.AdvanceGraph)"}[mode],
            "per_call": per_call,
        }
        emit_line(line)
    if d is not None:
        d.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the configuration's BASELINE step count, "
                         "cfg1 20, cfg2 100, cfg3 200, cfg4 50, cfg5 20)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="vpb", choices=["vpb", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20,
                    help="e2e steps (the pipeline fills once and drains once per call)")
    ap.add_argument("--e2e-blocks", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="replay the K timed steps from a CUDA graph (driver.AdvanceGraph; "
                         "with --per-step: per-step strang_step graphs, driver.StepGraph)")
    ap.add_argument("--per-step", action="store_true",
                    help="time one strang_step call per step instead of advance()")
    ap.add_argument("--layout", default="v", choices=["v", "x"],
                    help="N > 1, dG: v2 slabs (VShardedSolver, default) or x1 / x1 x x2 "
                         "shards (ShardedSolver)")
    ap.add_argument("--peer-halos", action="store_true",
                    help="--layout v: the v pass reads the neighbours' boundary rows in place "
                         "(CUDA IPC peer memory) instead of NCCL halo rows")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded multi-GPU solver (torch.distributed, NCCL) even at "
                         "N = 1: exercises the N > 1 code path on a one-GPU box")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas instead of the sharded field")
    ap.add_argument("--ref-budget", type=float, default=240.0,
                    help="--impl reference: seconds of timed full reference steps")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (from profiles/)")
    args = ap.parse_args()
    protect_stdout()
    if args.warmup < 3 and args.impl == "vpb":
        print("note: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.steps is None:
        args.steps = cfg["nsteps"]
    if args.impl == "reference":
        run_reference_arm(args, args.config, cfg)
    else:
        run_vpb(args, args.config, cfg)


if __name__ == "__main__":
    main()
