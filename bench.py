"""bench.py — DBFFT hot-path benchmark (driver contract).

Workload (BASELINE.json metric "voxel.CG-iter/s (fp64) and % HBM roofline at 256^3"):
config c4 — 256^3 finite-strain neo-Hookean two-phase composite (1202 RSA spheres of radius
10 voxels, vf 0.30, shear-modulus contrast 10, kappa/mu = 2.5), F_zz -> 1.10 in 10 increments,
P_xx = P_yy = 0 (mixed control).  One step = one load increment: the constitutive update,
residual, mean tangent and preconditioner, and Newton-PCG to tol_eq = 1e-10 / Newton 1e-6,
i.e. every row of SURVEY 8(a).  Steps walk the increments in order (state carried over);
after increment 10 the state is reset (inside the step that wraps).

value = voxels x PCG iterations / max-over-ranks device time, measured on the production path
(CUDA graphs with the device-side PCG loop, no per-kernel instrumentation).  Per-kernel times
(kernel_ms, the roofline of pass_X) come from a separate profiled pass of the next steps of the
walk (events around every launch, one PCG iteration per host poll so no launch is an early exit).
N > 1: the same c4 problem slab-decomposed over the N GPUs (z-slabs / ky-slabs, NCCL
all-to-all + all-reduce, or the peer transport; "scaling": "strong"); a rank that cannot build
its slab context fails the run (no silent fallback).  --replicas runs N independent copies.

--impl reference: the CPU oracle (oracle/dbfft_oracle.py) timed on this host: one oracle PCG
iteration (apply_K + preconditioner + CG algebra) of c4's first Newton step at 256^3 per step,
FFTs on all host cores.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxel*CG-iter/s (fp64), config c4 256^3"
UNIT = "voxel*iter/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(variant):
    """dram read+write bytes per launch of pass_X (this tangent variant) from the committed
    ncu --set full summary (profiles/ncu_pass_x_summary.json), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_pass_x_summary.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        v = d.get(variant)
        return v.get("dram_bytes_per_launch") if v else None
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return None
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows)}


# ------------------------------------------------------------------------------------------ GPU arm


# per-voxel material bytes read by pass_X at finite strain:
#   full    : 45 fp64 entries of the major-symmetric 9x9 tangent             = 360 B
#   compact : F^-1 (9 fp64) + c1 (1 fp64) + phase id (u16), tangent rebuilt  =  82 B
TANGENT_BYTES = {"full": 360, "compact": 82}


def bytes_pass_x(n, variant, kin=9):
    """Algorithmic bytes of one pass_X launch: c complex half-spectrum fields in and out
    (16 B each) plus the per-voxel tangent data of the variant in use."""
    n1, n2, n3 = n
    H = (n1 // 2 + 1) * n2 * n3
    N = n1 * n2 * n3
    return 2 * kin * 16 * H + TANGENT_BYTES[variant] * N


def bytes_apply_K(n, variant, kin=9):
    """Per-axis 5-pass schedule 16 * 66 * H + the variant's tangent bytes."""
    n1, n2, n3 = n
    H = (n1 // 2 + 1) * n2 * n3
    N = n1 * n2 * n3
    return 16 * (66 if kin == 9 else 52) * H + TANGENT_BYTES[variant] * N


def pcg_iteration_roofline(n, variant, t, iters, world, slab, peak):
    """SURVEY 8(d) "% HBM roofline of the full PCG iteration": the timed region's time per PCG
    iteration (Newton-step work — constitutive updates, true residuals — included) against
    B_iter = B_op + B_cg, the survey's per-axis model (full tangent, 480 H of CG vectors) at 8 TB/s,
    and against this schedule's algorithmic bytes (compact tangent; CG: 8 vector transfers of 48 H)
    at the measured copy peak.  Slabs: per GPU, the global bytes / world."""
    if not iters:
        return None
    n1, n2, n3 = n
    H = (n1 // 2 + 1) * n2 * n3
    t_it = t / (iters if slab or world == 1 else iters / world)  # one iteration of one problem
    share = world if slab else 1
    b_model = (bytes_apply_K(n, "full") + 480 * H) / share
    b_alg = (bytes_apply_K(n, variant) + 8 * 48 * H) / share
    return {"ms": t_it * 1e3, "survey_model_bytes": b_model, "survey_model_ms_8TBps": b_model / 8e12 * 1e3,
            "frac_of_survey_model": b_model / 8e12 / t_it, "algorithmic_bytes": b_alg,
            "achieved_GBps": b_alg / t_it / 1e9, "frac": b_alg / t_it / 1e9 / peak if peak else None}


def aggregate_over_ranks(t_local, iters, device="cuda"):
    """(max over ranks of the timed region, sum over ranks of the PCG iterations)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t_local, iters
    tt = torch.tensor([t_local], dtype=torch.float64, device=device)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    it = torch.tensor([float(iters)], dtype=torch.float64, device=device)
    dist.all_reduce(it, op=dist.ReduceOp.SUM)
    return float(tt.item()), int(round(it.item()))


def gpu_arm(args):
    import torch
    import torch.distributed as dist
    from paper_1905_12725_b200 import dbfft
    from synth import configs

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.c4(n=args.n, radius_vox=max(1, round(10 * args.n / 256)))
    n = cfg["n"]
    N = n[0] * n[1] * n[2]
    stream = torch.cuda.current_stream()
    mode = "single GPU"
    phase = cfg["phase"]
    if world > 1 and not args.replicas:
        # no fallback: a slab context that cannot be built (NCCL, peer windows) fails the run
        py = max(1, args.pencil_rows)
        ctx = dbfft.DBFFT(n, kinematics="finite", device=local, stream=stream, world=world, rank=rank,
                          transport=args.transport, pencil_rows=py)
        phase = rank_block(cfg["phase"], rank, world, py)
        pz = world // py
        if py > 1:
            mode = f"slab-pencils {py}x{pz} (2-D pencils, NCCL all-to-all in row / column groups + all-reduce)"
        else:
            mode = (f"slab x{world} (z-slabs / ky-slabs, " +
                    ("passes store into peer memory (VMM windows) + NCCL all-reduce)" if args.transport == "peer"
                     else "NCCL all-to-all + all-reduce)"))
    else:
        ctx = dbfft.DBFFT(n, kinematics="finite", device=local, stream=stream)
        if world > 1:
            mode = f"replicas x{world}"
    slab = mode.startswith("slab")
    ctx.set_phases(phase, cfg["materials"])
    # every rank logs its communicator view (device, rank / world, transport, NCCL comm) on stderr
    print(f"[dbfft rank {rank}/{world}] " + json.dumps(ctx.info()), file=sys.stderr, flush=True)
    loads = cfg["loads"]
    state = {"k": 0}

    def step():
        if state["k"] == len(loads):
            ctx.set_phases(phase, cfg["materials"])
            state["k"] = 0
        L = loads[state["k"]]
        rep = ctx.solve_increment(L["target"], L["mask"], dt=1.0, check_every=args.check_every)
        state["k"] += 1
        return rep

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ctx.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    iters = 0
    newton = 0
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            rep = step()
            iters += rep["cg_iters"]
            newton += rep["newton_iters"]
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - launches0
    pcg_loop = ctx.info()
    # per-kernel device times: a separate pass over the next steps of the walk with CUDA events
    # around every launch (graphs off, one PCG iteration per poll: no early-exit launches)
    prof_steps = max(1, min(args.steps, args.profile_steps))
    ctx.profile(True)
    prof_iters = 0
    for _ in range(prof_steps):
        prof_iters += step()["cg_iters"]
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    t_local = ms / 1e3
    t_max, tot_iters = aggregate_over_ranks(t_local, iters)
    if slab:  # one global problem: every rank counted the same iterations
        tot_iters = iters
    value = N * tot_iters / t_max

    # ------------------------------------------------ e2e: host inputs -> C ABI -> host result
    e2e = None
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    if e2e_steps > 0:
        # the same job through the public API from host memory: the microstructure is uploaded
        # from a pinned host map at the start of every load walk (set_phases), every increment
        # reads its load from the host and ends with the displacement field copied into a pinned
        # host buffer (allocated before the timed region, as a user reusing it would)
        import torch
        torch.cuda.synchronize()
        phase_host = torch.from_numpy(np.ascontiguousarray(phase, dtype=np.uint16).view(np.int16)).pin_memory().numpy().view(np.uint16)
        u_host = torch.empty((3,) + tuple(phase.shape), dtype=torch.float64, pin_memory=True).numpy()
        # untimed warm-up of the calls only this leg makes (the library's real-space scratch for
        # get_field is allocated on first use; lazily loaded kernels load on first launch)
        ctx.set_phases(phase_host, cfg["materials"])
        ctx.get_field(dbfft.FIELD_U, out=u_host)
        torch.cuda.synchronize()
        h2d = d2h = 0
        e_iters = 0
        k = 0
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            if k == 0:
                ctx.set_phases(phase_host, cfg["materials"])                  # H2D of the microstructure
                h2d += phase_host.nbytes
            L = loads[k]
            rep = ctx.solve_increment(L["target"], L["mask"], dt=1.0, check_every=args.check_every)
            h2d += 9 * 8 + 9                                                  # load target + mask
            ctx.get_field(dbfft.FIELD_U, out=u_host)                          # D2H of the displacement field
            d2h += u_host.nbytes + 2 * 9 * 8                                  # + macro strain / stress
            e_iters += rep["cg_iters"]
            k = (k + 1) % len(loads)
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        t_e2e_max, e_iters_tot = aggregate_over_ranks(t_e2e, e_iters)
        if slab:
            e_iters_tot = e_iters
        e2e = {"value": N * e_iters_tot / t_e2e_max, "unit": UNIT,
               "h2d_bytes_per_step": int(round(h2d / e2e_steps)), "d2h_bytes_per_step": int(round(d2h / e2e_steps)),
               "steps": e2e_steps, "cg_iters": e_iters,
               "note": "increments 1..K of the load walk through the C ABI: set_phases from a pinned host uint16 "
                       "map at the walk start, per increment the load from the host and get_field(U) into a "
                       "pinned host buffer; wall clock (max over ranks) around the calls"}
        # restore the walk state of the device-timed loop
        ctx.set_phases(phase, cfg["materials"])

    px_ms, px_n = prof.get("pass_X", (0.0, 0))
    peak, peak_src = measured_peaks()
    variant = "full" if os.environ.get("DBFFT_TANGENT") == "full" else "compact"
    bx = bytes_pass_x(n, variant)
    avg_x = px_ms / max(px_n, 1) / 1e3
    achieved = bx / avg_x / 1e9 if px_n else None
    # whole operator (all five passes) for context
    # the operator alone: inside the PCG the F3 pass also carries the fused residual update, so
    # apply_K is timed standalone (dbfft_apply_K on a random spectral vector, CUDA events)
    gen = torch.Generator(device="cuda").manual_seed(0)
    uh = ctx.empty_spectral()
    uh.copy_(torch.randn(uh.shape, dtype=torch.complex128, device=uh.device, generator=gen))
    fh = ctx.empty_spectral()
    for _ in range(2):
        ctx.apply_K(uh, fh)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_op = 10
    torch.cuda.synchronize()
    a0.record(stream)
    for _ in range(n_op):
        ctx.apply_K(uh, fh)
    a1.record(stream)
    torch.cuda.synchronize()
    op_ms = a0.elapsed_time(a1)
    del uh, fh
    op_gbs = bytes_apply_K(n, variant) / (op_ms / n_op / 1e3) / 1e9
    t_model = bytes_apply_K(n, "full") / 8e12  # SURVEY 8(d) model: 14.97 GB at 8 TB/s = 1.871 ms
    total_prof = sum(v[0] for v in prof.values())
    roofline = {"bound": "hbm", "kernel": f"pass_X (x C2R + neo-Hookean tangent contraction [{variant}] + R2C)",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": ncu_traffic(variant),
                "tangent": variant,
                "algorithmic_bytes_per_launch": bx, "avg_launch_ms": avg_x * 1e3, "launches": px_n,
                "peak_source": peak_src, "share_of_step": (px_ms / total_prof) if total_prof else None,
                "apply_K": {"measured": "standalone dbfft_apply_K x10 after the timed region (CUDA events)",
                            "algorithmic_bytes": bytes_apply_K(n, variant), "avg_ms": op_ms / n_op,
                            "achieved_GBps": op_gbs, "frac": (op_gbs / peak) if op_gbs else None,
                            "survey_model_ms_8TBps": t_model,
                            "frac_of_survey_model": t_model / (op_ms / n_op / 1e3)},
                "pcg_iteration": pcg_iteration_roofline(n, variant, t_max, tot_iters, world, slab, peak)}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
           "scaling": "strong" if slab else "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"c4: {n[0]}^3 finite-strain neo-Hookean, 30% RSA spheres r=10, "
                                  "F_zz->1.10 in 10 increments, P_xx=P_yy=0; one step = one increment",
                      "grid": list(n), "parallelism": mode,
                      "l2": "inputs larger than L2 (working set ~15 GB per GPU)", "tol_eq": 1e-10,
                      "tol_newton": 1e-6, "cg_iters_timed": iters, "newton_iters_timed": newton,
                      "pcg_loop": pcg_loop,
                      "timing": "value: CUDA events around the K steps on the production path (graphs, "
                                "no instrumentation); kernel_ms / roofline: a separate profiled pass of "
                                f"{prof_steps} further steps ({prof_iters} PCG iterations)"},
           "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches),
           "kernel_ms": {k: v[0] for k, v in prof.items()}}
    clk_sum = clk.summary()
    out["clocks"] = clk_sum
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        del ctx
        torch.cuda.empty_cache()
        out["cpu_baseline"] = cpu_baseline(args.cpu_n, reps=3)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------ oracle


def host_info():
    """Host cores, CPU model and memory (recorded with the oracle baseline)."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for line in f:
                k, v = line.split(":", 1)
                if k in ("MemTotal", "MemAvailable"):
                    info[k.lower() + "_gb"] = round(int(v.split()[0]) / 2 ** 20, 1)
    except OSError:
        pass
    return info


ORACLE_BYTES_PER_VOXEL = 1400  # full 3x3x3x3 tangent (648 B) + spectra / temporaries of one iteration


def oracle_grid(n_req):
    """Largest grid <= n_req whose oracle iteration fits the host memory (c4 at 256^3 needs ~24 GB)."""
    avail = host_info().get("memavailable_gb")
    n = n_req
    while avail is not None and n > 32 and n ** 3 * ORACLE_BYTES_PER_VOXEL > 0.8 * avail * 2 ** 30:
        n //= 2
    return n


def oracle_setup(n=256):
    """c4's first Newton step at grid n (the c4 phase map at n = 256): the tangent field at the
    first increment's homogeneous F, its mean, and the rhs b = F(div P) — oracle functions only."""
    from oracle import dbfft_oracle as O
    from synth import configs
    cfg = configs.c4(n=n, radius_vox=max(1, round(10 * n / 256)))
    ph = cfg["phase"]
    mu = np.array([m["mu"] for m in cfg["materials"]])[ph]
    kap = np.array([m["kappa"] for m in cfg["materials"]])[ph]
    L = cfg["loads"][0]
    F = np.where(L["mask"], np.eye(3), L["target"]).reshape(3, 3, 1, 1, 1) * np.ones((1, 1) + ph.shape)
    P, K = O.neo_hookean(F, mu, kap)
    del F, mu, kap
    XI = O.frequency_grid(cfg["n"])
    Kbar = O.volume_average(K)
    b = O.rhs_from_stress(P, XI)
    return dict(O=O, K=K, XI=XI, Kbar=Kbar, b=b, mask=L["mask"], N=ph.size, n=cfg["n"])


def oracle_iteration(S, p, r, rz):
    """One PCG iteration of the oracle (apply_K + preconditioner + CG algebra), as in O.pcg."""
    O = S["O"]
    q, _ = O.apply_K(p, S["K"], S["XI"], finite=True)
    alpha = rz / O.inner(p, q)
    r = r - alpha * q
    z = O.precondition(r, S["Kbar"], S["XI"])
    rz_new = O.inner(r, z)
    p = z + (rz_new / rz) * p
    return p, r, rz_new


def oracle_start(S):
    O = S["O"]
    r = S["b"]
    z = O.precondition(r, S["Kbar"], S["XI"])
    return z, r, O.inner(r, z)


def oracle_sample_text(n, what):
    from oracle import dbfft_oracle as O
    return (f"{what} of c4's first Newton step at {n}^3 (c4's phase map, full 3x3x3x3 tangent, full complex "
            f"spectra): apply_K + preconditioner + CG algebra; scipy.fft on {O.FFT_WORKERS} threads, the rest "
            "numpy on one thread")


def cpu_baseline(n_req=256, reps=3):
    """The oracle as it stands on this host: median over `reps` PCG iterations at c4's grid."""
    n = oracle_grid(n_req)
    from oracle import dbfft_oracle as O
    S = oracle_setup(n)
    p, r, rz = oracle_start(S)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        p, r, rz = oracle_iteration(S, p, r, rz)
        times.append(time.perf_counter() - t0)
    t = float(np.median(times))
    what = f"median of {reps} oracle PCG iterations"
    if n != n_req:
        what += f" (host memory too small for {n_req}^3: measured at {n}^3)"
    return {"value": S["N"] / t, "unit": UNIT, "cores": O.FFT_WORKERS, "kind": "oracle",
            "sample": oracle_sample_text(n, what), "seconds_per_iteration": t, "iterations": times,
            "grid": [n] * 3, "host": host_info()}


def reference_arm(args):
    """The oracle (this tier's reference) on the bench's metric and workload: one oracle PCG
    iteration of c4 at 256^3 per step (one warm-up iteration: the oracle has no state to warm)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n = oracle_grid(args.cpu_n)
    from oracle import dbfft_oracle as O
    S = oracle_setup(n)
    p, r, rz = oracle_start(S)
    for _ in range(min(args.warmup, 1)):
        p, r, rz = oracle_iteration(S, p, r, rz)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        p, r, rz = oracle_iteration(S, p, r, rz)
    t = time.perf_counter() - t0
    v = S["N"] * args.steps / t
    sample = oracle_sample_text(n, "one oracle PCG iteration per step")
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic",
                      "config": {"workload": f"c4: {n}^3 finite-strain neo-Hookean (oracle, first Newton step)",
                                 "grid": [n] * 3, "host": host_info()},
                      "cpu_baseline": {"value": v, "unit": UNIT, "cores": O.FFT_WORKERS, "kind": "oracle",
                                       "sample": sample},
                      "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def rank_block(field, rank, world, py=1):
    """This rank's real-space block [z][y][x] of a global field (include/dbfft.h: rank = b Py + a
    owns z in [b n3/Pz, ...) x y in [a n2/Py, ...), all x; Py = 1: z-slabs)."""
    pz = world // py
    n3, n2 = field.shape[-3], field.shape[-2]
    nzl, nyr = n3 // pz, n2 // py
    a, b = rank % py, rank // py
    return np.ascontiguousarray(field[..., b * nzl:(b + 1) * nzl, a * nyr:(a + 1) * nyr, :])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dbfft", choices=["dbfft", "reference"])
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--check-every", type=int, default=8)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-n", type=int, default=256, help="grid of the oracle baseline (c4 at 256^3)")
    ap.add_argument("--profile-steps", type=int, default=2, help="steps of the separate per-kernel profiled pass")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of slabs")
    ap.add_argument("--pencil-rows", type=int, default=1,
                    help="N > 1: 2-D pencil decomposition on a Py x (N / Py) grid (default 1: z-slabs)")
    ap.add_argument("--transport", choices=("nccl", "peer"), default="nccl",
                    help="N > 1 slabs: NCCL all-to-all exchanges, or passes storing into peer memory")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
