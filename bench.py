#!/usr/bin/env python3
"""Benchmark of the B200 mod-p SYRK hot path (metric of BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

A "step" is one full call of the hot path on one input of the chosen config
(default cfg2 = configs[1]: p = 131071, A 4096 x 4096, recursion to 512-leaves).
`value` is effective n^2 k / t (GOPS) over device-resident inputs (CUDA
events on the launching stream, L2 flushed between steps); `e2e` is the same
metric through the host C-ABI entry point from the caller's pageable numpy
buffers (`e2e_pinned`: from pinned buffers).
N > 1 ranks: launched by torchrun (one process per GPU), or by this script itself
when `--gpus N` is given without WORLD_SIZE in the environment.  Default
`--mgpu partition`: the ranks split one problem's top-level tile pairs (strong
scaling); `--mgpu replicas`: one independent problem per rank (weak
scaling).  The timed region is bracketed by barriers and the max over ranks is
reported.  `--impl reference` times the reference's own CPU implementation
(oracle/_ref/ref_driver, built from the reference sources) on the host cores.
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

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

UNL = (1 << 64) - 1
CONFIGS = {
    # name: p, n, k, seed, threshold, max_levels, mode  (BASELINE.json "configs", in order)
    "cfg1": dict(p=65537, n=1024, k=1024, seed=42, threshold=64, levels=1, mode="plain"),
    "cfg2": dict(p=131071, n=4096, k=4096, seed=42, threshold=1024, levels=UNL, mode="plain"),
    # configs 3-5 leave the recursion depth to the builder: the policy below is the fastest
    # measured depth (>= 1 level; profiles/r01/policy_sweep.txt) -- the result does not depend on it
    "cfg3": dict(p=65521, n=8192, k=2048, seed=42, threshold=2, levels=1, mode="acc", cseed=43, abseed=7),
    "cfg4": dict(p=2147483647, n=16384, k=16384, seed=42, threshold=2, levels=2, mode="plain"),
    "cfg5": dict(p=131071, n=32768, k=1024, seed=5001, threshold=2, levels=1, mode="schur", cseed=5003,
                 dseed=5002),
}
METRIC = "mod-p SYRK C=AAᵀ effective GOPS (n²k/t) at 1–8 B200; % of tensor-core peak"
# CPU samples of the reference (cpu_baseline leg and --impl reference): configs 1-2 run the
# config itself (n = k = 4096 for cfg2: ~25-35 s per single-threaded call); configs 3-5 take
# 1-25 min per call single-threaded, so they run a bounded sample (same prime / mode / leaf size,
# smaller n) and say so in the line's `sample` and `same_config: false`
CPU_SAMPLE = {
    "cfg1": dict(n=1024, k=1024, threshold=64, levels="1"),
    "cfg2": dict(n=4096, k=4096, threshold=1024, levels="inf"),
    "cfg3": dict(n=2048, k=512, threshold=512, levels="inf"),
    "cfg4": dict(n=2048, k=2048, threshold=512, levels="inf"),
    "cfg5": dict(n=4096, k=256, threshold=512, levels="inf"),
}
# the reference arm's warm-up waves: a 64x smaller instance of the same prime and policy (a warm-up
# only pages in the binary and settles the host clocks; a full cfg2 wave is ~30 s)
CPU_WARM = dict(n=1024, k=1024)


def same_config(cfgname, cfg):
    s = CPU_SAMPLE[cfgname]
    return s["n"] == cfg["n"] and s["k"] == cfg["k"]


def load_peaks():
    peaks = {}
    try:
        peaks.update(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))))
    except Exception:
        pass
    try:
        peaks.update(json.load(open(os.path.join(REPO, "profiles", "int8_peak.json"))))
    except Exception:
        pass
    return peaks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FSYRK_B200_BENCH_PART1=1: run the multi-GPU partition path as a single rank (one-GPU test
    # of its NCCL / staging plumbing; the result is the single-GPU problem)
    if world > 1 or os.environ.get("FSYRK_B200_BENCH_PART1"):
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def cpu_reference(cfgname, cfg, threads, reps=1, sample=None):
    """Run the unmodified reference (oracle/_ref/ref_driver): `threads` concurrent independent
    instances of the sample (default CPU_SAMPLE[cfgname]), each `reps` calls."""
    drv = os.path.join(REPO, "oracle", "_ref", "ref_driver")
    if not os.path.exists(drv):
        return None
    s = dict(CPU_SAMPLE[cfgname])
    if sample:
        s.update(sample)
    cmd = [drv, "--p", str(cfg["p"]), "--n", str(s["n"]), "--k", str(s["k"]), "--seed", str(cfg["seed"]),
           "--threshold", str(s["threshold"]), "--levels", s["levels"], "--mode", cfg["mode"],
           "--threads", str(threads), "--reps", str(reps), "--no-digest"]
    if "cseed" in cfg:
        cmd += ["--cseed", str(cfg["cseed"])]
    if "abseed" in cfg:
        cmd += ["--abseed", str(cfg["abseed"])]
    if "dseed" in cfg:
        cmd += ["--dseed", str(cfg["dseed"])]
    out = json.loads(subprocess.run(cmd, check=True, capture_output=True, text=True).stdout)
    e = float(s["n"]) ** 2 * float(s["k"])
    gops = e * threads * reps / out["wall_seconds"] / 1e9
    return {"value": round(gops, 4), "unit": "GOPS", "cores": threads, "kind": "reference",
            "sample": f"reference syrk ({cfg['mode']}) p={cfg['p']} n={s['n']} k={s['k']} threshold={s['threshold']}"
                      f" levels={s['levels']}, {threads} concurrent instance(s) x {reps}",
            "same_config": s["n"] == cfg["n"] and s["k"] == cfg["k"],
            "seconds": out["wall_seconds"]}


def cpu_reference_bounded(cfgname, cfg, target_s=10.0):
    """The reference on one core (the cpu_baseline leg, timed on the box's own host): one call of
    the config itself when that is cfg1 / cfg2 (cfg2: ~25-35 s), else the bounded sample repeated
    to about target_s seconds of CPU work."""
    first = cpu_reference(cfgname, cfg, 1, 1)
    if first is None or first["same_config"]:
        return first
    reps = max(1, min(50, int(target_s / max(first["seconds"], 1e-3) + 0.5)))
    return cpu_reference(cfgname, cfg, 1, reps) if reps > 1 else first


def run_reference(args, cfgname, cfg, world, rank):
    """--impl reference: the reference's own CPU implementation on all host cores, one
    independent single-threaded instance per core (the reference has no threaded mode,
    proj/README.md:149); a step is one wave of those instances on the config (cfg1 / cfg2:
    the config itself, e.g. 16 x cfg2 per ~30 s step)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if not os.path.exists(os.path.join(REPO, "oracle", "_ref", "ref_driver")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_driver not built"}))
        return
    for _ in range(args.warmup):
        cpu_reference(cfgname, cfg, threads, reps=1, sample=CPU_WARM)
    budget = float(os.environ.get("FSYRK_B200_REF_BUDGET_S", "1500"))
    times, base = [], None
    t_start = time.perf_counter()
    for i in range(args.steps):
        r = cpu_reference(cfgname, cfg, threads, reps=1)
        base = base or r
        times.append(r["seconds"])
        # stay inside the driver's per-command limit: stop once the next wave would not fit
        if (time.perf_counter() - t_start) * (i + 2) / (i + 1) > budget:
            break
    s = CPU_SAMPLE[cfgname]
    e = float(s["n"]) ** 2 * float(s["k"]) * threads
    total = sum(times)
    value = e * len(times) / total / 1e9
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GOPS", "n_gpus": max(world, args.gpus),
            "steps": len(times), "steps_requested": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total / len(times) * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (reference random_matrix)",
            "impl": "reference",
            "config": {"workload": cfgname, **{k: v for k, v in cfg.items() if k != "levels"},
                       "levels": "inf" if cfg["levels"] == UNL else cfg["levels"], "sample": base["sample"],
                       "warmup_sample": f"n={CPU_WARM['n']} k={CPU_WARM['k']}"},
            "vs_reference": {"same_config": base["same_config"]},
            "cpu_baseline": {"value": round(value, 4), "unit": "GOPS", "cores": threads, "kind": "reference",
                             "sample": base["sample"], "same_config": base["same_config"]},
            "e2e": {"value": round(value, 4), "unit": "GOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def spawn_ranks(ngpus):
    """`--gpus N` without a launcher: start N ranks (one process per GPU) with torchrun on this
    node and pass rank 0's JSON line through.  NCCL_DEBUG=INFO stays on so every rank's NCCL
    init is visible in the log."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < ngpus:
        print(f"bench.py: --gpus {ngpus} requested but only {have} CUDA device(s) are visible", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def max_over_ranks(value, world):
    """Max of a per-rank scalar over all ranks (device timing rule: the slowest rank counts)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def lower_digest(c):
    import hashlib
    h = hashlib.sha256()
    for i in range(c.shape[0]):
        h.update(np.ascontiguousarray(c[i, : i + 1]).astype("<u8").tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mgpu", default="partition", choices=["partition", "replicas"],
                    help="N > 1: split one problem's top level across ranks (strong scaling) or run one "
                         "independent problem per rank (weak scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--threshold", type=int, default=None, help="override the config's recursion threshold")
    ap.add_argument("--levels", type=int, default=None, help="override the config's max recursion levels")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    cfg = dict(CONFIGS[args.config])
    if args.threshold is not None:
        cfg["threshold"] = args.threshold
    if args.levels is not None:
        cfg["levels"] = args.levels
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, args.config, cfg, world, rank)
        return

    import torch
    import paper_2001_04109_b200 as fs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    part = (world > 1 or bool(os.environ.get("FSYRK_B200_BENCH_PART1"))) and args.mgpu == "partition"
    if world > 1 or part:
        import torch.distributed as dist
    p, n, k = cfg["p"], cfg["n"], cfg["k"]
    f = fs.PrimeField(p)
    policy = fs.RecursionPolicy(cfg["threshold"], cfg["levels"])
    seed = cfg["seed"] + (0 if part else rank)  # partition: one problem; replicas: one per rank
    a_host = fs.random_matrix(f, n, k, seed)
    alpha, beta, d = 1, 0, None
    c0_host = None
    if cfg["mode"] in ("acc", "schur"):
        c0_host = fs.random_matrix(f, n, n, cfg["cseed"])
        iu = np.triu_indices(n, 1)
        c0_host[iu] = c0_host.T[iu]
    if cfg["mode"] == "acc":
        # alpha, beta = 1 + rng() % (p-1) from mt19937_64(abseed) (oracle/ref_driver.cpp convention)
        alpha, beta = _mt_alpha_beta(p, cfg["abseed"])
    if cfg["mode"] == "schur":
        d = _mt_nonzero(p, k, cfg["dseed"])
        alpha, beta = p - 1, 1

    a_dev = torch.from_numpy(a_host.view(np.int64)).to(dev)
    c_dev = torch.zeros((n, n), dtype=torch.int64, device=dev)
    c_init = torch.from_numpy(c0_host.view(np.int64)).to(dev) if c0_host is not None else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step():
        if part:
            fs.syrk_part_dev(p, alpha, a_dev.data_ptr(), n, k, k, beta, c_dev.data_ptr(), n, policy, rank, world, sh,
                             d=d)
        else:
            fs.syrk_dev(p, alpha, a_dev.data_ptr(), n, k, k, beta, c_dev.data_ptr(), n, policy, False, sh, d=d)

    def reset_c():
        if c_init is not None:
            c_dev.copy_(c_init)
        elif part:
            c_dev.zero_()

    # warm-up (plan creation happens on the first call)
    for _ in range(max(args.warmup, 3)):
        reset_c()
        step()
    torch.cuda.synchronize()
    launches = fs.last_launch_counts()
    plan = fs.last_plan()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # the timed region is milliseconds long: keep the GPU busy with the same step until the
        # sampler reports, so the clock record covers the load the timed steps run under
        t_end = time.time() + 3.0
        while time.time() < t_end and len(clk.samples) < 3:
            for _ in range(20):
                reset_c()
                step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()
        for i in range(args.steps):
            reset_c()
            flush.zero_()
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        clk.samples = list(clk.samples)  # samples up to the end of the timed region only
    if world > 1:
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms_max = max_over_ranks(ms, world)
    E = float(n) * n * k
    problems = 1 if part else world
    value = E * args.steps * problems / (ms_max / 1e3) / 1e9

    # parity self-check of the device output against the reference's digest of the config
    parity = None
    ref_json = os.path.join(REPO, "tests", "golden", "configs", f"{args.config}.json")
    ref_digest = json.loads(open(ref_json).read())["digest"] if os.path.exists(ref_json) else None
    comm = None
    comm_error = None
    if part:  # the library's multi-GPU call: NCCL communicator from a unique id made on rank 0
        try:
            obj = [fs.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            comm = fs.Communicator(obj[0], rank, world)
        except Exception as ex:  # noqa: BLE001  (the device-timed value above stands on its own)
            comm_error = f"{type(ex).__name__}: {ex}"
            comm = None
    if ref_digest and not part:
        try:
            reset_c()
            step()
            torch.cuda.synchronize()
            parity = "digest-match" if lower_digest(c_dev.cpu().numpy().view(np.uint64)) == ref_digest \
                else "DIGEST-MISMATCH"
        except Exception as ex:  # noqa: BLE001
            parity = f"unchecked ({type(ex).__name__})"
    elif ref_digest and comm is not None:  # partitioned: the whole multi-GPU call on the host C
        try:
            c_chk = c0_host.copy() if c0_host is not None else np.zeros((n, n), dtype=np.uint64)
            plan_chk = fs.make_syrk_plan(f, policy)
            comm.syrk(f, a_host if rank == 0 else None, c_chk if rank == 0 else None, n, k, plan_chk, alpha, beta, d)
            if rank == 0:
                parity = "digest-match" if lower_digest(c_chk) == ref_digest else "DIGEST-MISMATCH"
        except Exception as ex:  # noqa: BLE001
            parity = f"unchecked ({type(ex).__name__}: {ex})"

    # per-phase device times (phase events inside the library, same stream) for the roofline
    fs.set_phase_timing(True)
    phase = {"products": 0.0, "pre": 0.0, "post": 0.0, "convert": 0.0}
    reps = max(3, min(args.steps, 10))
    for _ in range(reps):
        reset_c()
        flush.zero_()
        step()
        for key, v in fs.last_phase_ms().items():
            phase[key] += v / reps
    fs.set_phase_timing(False)
    torch.cuda.synchronize()

    # end-to-end through the public API: host A -> device(s) -> host Low(C).  Default: pageable
    # numpy buffers, the memory a drop-in caller hands in (the reference's Matrix is a
    # std::vector, matrix.hpp:122-126); the same from pinned buffers is reported beside it.
    e2e = e2e_pinned = None
    if not args.no_e2e:
        plan_obj = fs.make_syrk_plan(f, policy)

        def measure(a_np, c_np):
            if cfg["mode"] != "plain":
                c_np[:] = c0_host

            def host_step():
                if part:  # the library's collective multi-GPU call: rank 0 holds the host A and C
                    comm.syrk(f, a_np if rank == 0 else None, c_np if rank == 0 else None, n, k, plan_obj, alpha,
                              beta, d)
                elif cfg["mode"] == "plain":
                    fs.syrk_fast_into(f, a_np, c_np, plan_obj)
                elif cfg["mode"] == "acc":  # C accumulates across steps (any C_in is a valid input)
                    fs.syrk_fast_acc(f, alpha, a_np, beta, c_np, plan_obj)
                else:
                    fs.syrkd(f, a_np, d, plan_obj, alpha=alpha, beta=beta, c=c_np)

            for _ in range(6):  # warm-up (also lets host_io settle its raw-DMA shares)
                host_step()
            e2e_steps = max(3, min(args.steps, 10))
            # three timed rounds of e2e_steps calls, the median round reported: the host side of the
            # transfers is sensitive to host-CPU noise (e.g. right after an all-core CPU run)
            round_secs = []
            for _ in range(3):
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                for _ in range(e2e_steps):
                    host_step()
                t1 = time.perf_counter()
                round_secs.append(max_over_ranks(t1 - t0, world))
            secs = statistics.median(round_secs)
            # what the host API moved (A, and the lower-triangle row blocks of C); partitioned: rank
            # 0's PCIe traffic (the NVLink broadcast / share gather are device-to-device)
            h2d, d2h = fs.last_transfer_bytes()
            if not part:
                h2d, d2h = h2d * world, d2h * world
            return {"value": round(E * e2e_steps * problems / secs / 1e9, 3), "unit": "GOPS",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

        if part and comm is None:
            e2e = {"unavailable": f"NCCL communicator: {comm_error}"}
        else:
            try:
                # pageable (the default e2e): the numpy arrays the caller owns
                e2e = measure(np.ascontiguousarray(a_host), np.zeros((n, n), dtype=np.uint64))
                e2e["host_memory"] = "pageable"
                a_pin = torch.from_numpy(a_host.view(np.int64)).pin_memory()
                c_pin = torch.zeros((n, n), dtype=torch.int64).pin_memory()
                e2e_pinned = measure(a_pin.numpy().view(np.uint64), c_pin.numpy().view(np.uint64))
                e2e_pinned["host_memory"] = "pinned"
            except Exception as ex:  # noqa: BLE001
                e2e = e2e or {"unavailable": f"{type(ex).__name__}: {ex}"}

    if comm is not None:
        comm.close()
    if rank != 0:
        if world > 1 or part:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    # algorithmic int8 ops: 2 x (distinct digit-plane products per modular MAC) x modular MACs
    int8_ops = 2.0 * plan.get("terms", 9) * plan.get("tensor_macs", 0)
    nprod = max(1, launches.get("products", 1))
    prod_ms = phase["products"]
    peak_i8 = peaks.get("int8_tops")
    peak_src = "measured int8 (torch._int_mm, profiles/int8_peak.json)"
    if not peak_i8:
        peak_i8 = 2.0 * peaks.get("bf16_tflops", 1590.0)
        peak_src = "2 x measured bf16 (MEASURED_PEAKS.json)"
    achieved = int8_ops / (prod_ms / 1e3) / 1e12 if prod_ms > 0 else 0.0
    traffic = None
    try:
        traffic = json.load(open(os.path.join(REPO, "profiles", "traffic.json"))).get(args.config)
    except Exception:  # noqa: BLE001
        pass
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(peak_i8, 1), "unit": "TFLOP/s",
                "frac": round(achieved / peak_i8, 4) if peak_i8 else None, "traffic": traffic,
                "kernel": "modmm (tcgen05 kind::i8 limb products)", "launches_per_step": nprod,
                "avg_launch_ms": round(prod_ms / nprod, 4), "peak_source": peak_src,
                "algorithmic_int8_ops_per_step": int8_ops, "rank": 0,
                # ncu's int8 tensor peak: 16384 ops/clk/SM x 148 SMs x 1.965 GHz
                "nominal_peak": 4765.4, "nominal_frac": round(achieved / 4765.4, 4),
                "phase_ms": {k2: round(v, 4) for k2, v in phase.items()}}
    # the elementwise phases against HBM: algorithmic bytes (plan JSON, driver.cu) / phase time
    hbm_peak = peaks.get("hbm_gbs")
    post_b = plan.get("post_bytes", 0) + (plan.get("post_cin_bytes", 0) if beta % p else 0)
    hbm = {}
    for key, nbytes in (("convert", plan.get("convert_bytes", 0)), ("pre", plan.get("prep_bytes", 0)),
                        ("post", post_b)):
        t = phase.get(key, 0.0)
        if t > 0 and nbytes:
            gbs = nbytes / (t / 1e3) / 1e9
            hbm[key] = {"algorithmic_bytes": nbytes, "ms": round(t, 4), "achieved": round(gbs, 1),
                        "frac": round(gbs / hbm_peak, 4) if hbm_peak else None}
    roofline["elementwise_hbm"] = {"peak": hbm_peak, "unit": "GB/s",
                                   "peak_source": "measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs)", **hbm}
    cpu = None if (args.no_cpu_baseline or world > 1) else cpu_reference_bounded(args.config, cfg)
    if cpu is not None:
        cpu.pop("seconds", None)
    clocks = clk.summary()
    line = {"metric": METRIC, "value": round(value, 2), "unit": "GOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if part else "weak", "vs_baseline": None,
            "dtype": "int8",  # tensor-core digit products (int32 accumulate); uint32 residues elsewhere
            "dtype_detail": "int8 digit planes x int8 -> int32 TMEM accumulators; uint32 mod-p residues in the "
                            "elementwise kernels; uint64 at the API boundary",
            "data": "synthetic (reference random_matrix stream)",
            "config": {"workload": args.config, "p": p, "n": n, "k": k, "mode": cfg["mode"],
                       "threshold": cfg["threshold"], "levels": "inf" if cfg["levels"] == UNL else cfg["levels"],
                       "parallelism": (f"top-level tile-pair partition x{world}" if part else f"replicas x{world}"),
                       "l2": "flushed between steps (256 MiB write)"},
            "parity": parity, "gpu_launches": launches["total"] * args.steps,
            "launches_per_step": launches, "roofline": roofline, "cpu_baseline": cpu,
            "vs_reference": {"same_config": bool(cpu and cpu.get("same_config")),
                             "reference_sample": cpu and cpu.get("sample")},
            "e2e": e2e, "e2e_pinned": e2e_pinned,
            "clocks": clocks, "plan": {k2: plan.get(k2) for k2 in ("scheme", "terms", "block_n", "nodes", "leaf_groups",
                                                                     "gemm_groups", "arena_bytes", "schedule", "tree_prep",
                                                                     "winograd_groups")}}
    print(json.dumps(line))
    if world > 1 or part:
        dist.destroy_process_group()


def _mt_alpha_beta(p, seed):
    """alpha, beta = 1 + rng() % (p - 1) from std::mt19937_64(seed)."""
    x = _mt64(seed, 2)
    return 1 + int(x[0]) % (p - 1), 1 + int(x[1]) % (p - 1)


def _mt_nonzero(p, count, seed):
    """D = 1 + rng() % (p - 1) from mt19937_64(seed) (oracle/ref_driver.cpp make_instance;
    BASELINE.md's config-5 convention: seeds 5001/5002/5003 give 526 non-residues)."""
    return np.array([1 + int(x) % (p - 1) for x in _mt64(seed, count)], dtype=np.uint64)


def _mt64(seed, count):
    mt = [0] * 312
    mt[0] = seed & ((1 << 64) - 1)
    for i in range(1, 312):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & ((1 << 64) - 1)
    idx = 312
    out = []
    for _ in range(count):
        if idx >= 312:
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            idx = 0
        z = mt[idx]
        idx += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000
        z ^= (z << 37) & 0xFFF7EEE000000000
        z ^= z >> 43
        out.append(z & ((1 << 64) - 1))
    return np.array(out, dtype=np.uint64)


if __name__ == "__main__":
    main()
