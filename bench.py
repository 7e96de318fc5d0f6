"""Benchmark of the hot path: FP64 two-site H_eff.psi inside Lanczos, at C4 (m = 4096).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl heff|reference]

A step is one Lanczos iteration through the C ABI (lanczos_ground, fixed-step mode):
one H_eff.psi matvec (GEMM1 L.psi -> fused MPO W1.W2 -> GEMM4 .R^T; at N > 1 order B
on a b'-shard plus the NCCL all-gather of psi), CGS2 reorthogonalisation, the norm and
the host tridiagonal solve.  value = matvecs/s of the whole job (strong scaling: one
fixed m = 4096 problem split over N GPUs).  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, plain C loops, all host cores) on a
bounded sample of the same workload (rows a' of the output), rank 0 only.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "H_eff·ψ matvecs/s and FP64 TFLOP/s vs B200 FP64 peak at m=4096, 1/2/4/8 GPU"
# FP64 peak: 148 SM x 128 flop/clk/SM x 1.965 GHz; the DMMA microbenchmark measured 37.16 TF/s
# sustained at 1965 MHz (profiles/r01_fp64_peaks.txt).  MEASURED_PEAKS.json has no FP64 entry.
FP64_PEAK_TFLOPS = 148 * 128 * 1.965e9 / 1e12


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class Clocks:
    """nvidia-smi sampler for the timed region (clocks + throttle reasons)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        pw = [float(r[2]) for r in self.rows if len(r) >= 7 and r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "power_w_max": max(pw) if pw else None}


def workload_name(cfg: str, dims: dict) -> str:
    model = {"c1": "heisenberg_chain", "c2": "heisenberg_chain", "c3": "heisenberg_chain", "c4": "cylinder6",
             "c5": "hubbard"}[cfg]
    return f"{cfg}_{model}_m{dims['mL']}_d{dims['d1']}_k{dims['kL']}"


def cpu_baseline(x, budget_s: float = 12.0) -> dict:
    """The oracle as it stands, on rows a' of the same C4 inputs, for ~budget_s seconds."""
    from oracle import oracle
    oracle.build()
    L, W1, W2, R, psi = x.numpy()
    mL = L.shape[0]
    cores = oracle.max_threads()
    rows_done, t0 = 0, time.perf_counter()
    while True:
        lo = rows_done % mL
        hi = min(mL, lo + cores)
        oracle.heff_apply(L, W1, W2, R, psi, rows=(lo, hi))
        rows_done += hi - lo
        el = time.perf_counter() - t0
        if el >= budget_s or rows_done >= mL:
            break
    return {"value": rows_done / mL / el, "unit": "matvec/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{rows_done} of {mL} output rows a' (order A, independent per a'), {el:.1f} s; "
                      f"value = rows/s / mL", "seconds": el}


def bench_config(cfg: str, dims: dict, flops: float) -> dict:
    """The workload description both arms print (identical dicts: same metric, same config)."""
    return {"workload": workload_name(cfg, dims), **dims, "flops_per_matvec": flops,
            "step": "one Lanczos iteration (one H_eff.psi matvec + CGS2 + norm + host tridiagonal)",
            "l2": "inputs larger than L2 (psi 0.54 GB, L and R 2.7 GB each)" if cfg == "c4" else "see DESIGN.md 7"}


def run_reference(args):
    """--impl reference: the CPU oracle timed on bounded samples of the same workload.

    Each step computes a bounded sample of one matvec -- `cores` output rows a' (order A
    rows are independent), one per host thread -- and its measured wall time is the line's
    ms_per_step; value (matvec/s) = (rows / mL) / that time.  The whole-matvec time this
    implies is reported separately (ms_per_matvec_extrapolated), checked against one whole
    oracle matvec in profiles/r02_oracle_timings.json."""
    import numpy as np  # noqa: F401
    import torch
    from heffgen import configs as C
    from oracle import oracle

    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    oracle.build()
    # all host cores (torchrun exports OMP_NUM_THREADS=1 to its ranks; only rank 0 works here)
    oracle.set_threads(os.cpu_count() or 1)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    x = C.make(args.config, device=dev).to("cpu")
    L, W1, W2, R, psi = x.numpy()
    mL = L.shape[0]
    cores = oracle.max_threads()
    rows = cores  # one row per thread per step
    for _ in range(args.warmup):
        oracle.heff_apply(L, W1, W2, R, psi, rows=(0, rows))
    t0 = time.perf_counter()
    for s in range(args.steps):
        lo = (s * rows) % mL
        oracle.heff_apply(L, W1, W2, R, psi, rows=(lo, min(mL, lo + rows)))
    el = time.perf_counter() - t0
    frac = rows / mL
    value = args.steps * frac / el
    flops = C.flops_per_matvec(x.dims)
    sample = f"each step = {rows} of {mL} output rows a' of one matvec (order A oracle, one row per thread)"
    line = {"metric": METRIC, "value": value, "unit": "matvec/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "ms_per_matvec_extrapolated": el / args.steps * 1e3 / frac,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.config, x.dims, flops), "layout": "CPU oracle (oracle/heff_oracle.c, OpenMP)",
            "tflops": value * flops / 1e12,
            "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_model() -> str | None:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def dry_run(args) -> int:
    """--dry-run: the rank plumbing alone (gloo on CPU): every rank joins, the ranks are summed."""
    import torch
    import torch.distributed as dist
    world = env_int("WORLD_SIZE", 1)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
        return 2
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.tensor([float(env_int("RANK", 0))])
        dist.all_reduce(t)
        dist.destroy_process_group()
        total = int(t.item())
    else:
        total = 0
    if env_int("RANK", 0) == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "rank_sum": total}), flush=True)
    return 0


def spawn_ranks(n: int, check_devices: bool = True) -> int:
    """--gpus N without a torchrun environment: re-launch this command as N ranks (one per
    GPU) under torch.distributed.run and return its exit code.  Fewer than N visible GPUs is
    an error (never a 1-GPU number labelled as N)."""
    import torch
    have = torch.cuda.device_count()
    if check_devices and have < n:
        print(f"bench.py: --gpus {n} but only {have} CUDA device(s) are visible", file=sys.stderr)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    print("bench.py: spawning " + " ".join(cmd[1:6]) + f" ... ({n} ranks)", file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def load_ncu_traffic(kernel_key: str):
    """DRAM bytes per launch of the dominant kernel from one `ncu --set full` capture
    (profiles/ncu_summary.json, written by tools/ncu_summarize.py) and where they come from."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None, None
    try:
        e = json.loads(f.read_text()).get(kernel_key, {})
        src = f"profiles/{e.get('tag')}_ncu.md (ncu --set full, build of commit {e.get('commit')})" if e else None
        return e.get("dram_bytes_per_launch"), src
    except Exception:
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="heff", choices=["heff", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--sharded", action="store_true",
                    help="use the b'-sharded NCCL plan even at N=1 (exercises the multi-GPU code path)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check only: spawn the N ranks (gloo, no GPU work), all-reduce their ranks and "
                         "print one JSON line from rank 0")
    ap.add_argument("--fused-gather", action="store_true",
                    help="sharded plans: GEMM_A reads the ranks' Krylov shards through NCCL symmetric-window "
                         "(NVLink) pointers instead of ncclAllGather + relayout (NEXT-5)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus < 1:
        print("bench.py: --gpus must be >= 1", file=sys.stderr)
        return 2
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus, check_devices=not args.dry_run)
    if args.dry_run:
        return dry_run(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from heffgen import configs as C
    from paper_2007_14822_b200 import Heff
    from paper_2007_14822_b200 import dist as hdist
    from paper_2007_14822_b200.heff import (OPT_FUSED_GATHER, OPT_LANCZOS_RESERVE, OPT_PROFILE, OPT_TOTAL_LAUNCHES,
                                              nccl_unique_id)

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}: refusing to report a mismatched n_gpus",
              file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.sharded
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)

    # ---- inputs (seeded, synthetic; generated on the GPU, then broadcast from rank 0)
    x = C.make(args.config, device=dev)
    dims = x.dims
    if sharded:
        for t in (x.L, x.W1, x.W2, x.R, x.psi):
            dist.broadcast(t, 0)
    mR = dims["mR"]
    flops = C.flops_per_matvec(dims)
    gemm_flops = C.gemm_flops_per_matvec(dims)
    if sharded:
        lo, hi = hdist.shard_range(mR, world, rank)
        uid = hdist.broadcast_uid(nccl_unique_id() if rank == 0 else None, device=dev)
        Rg = x.R[lo:hi].contiguous()
        plan = Heff(x.L, x.W1, x.W2, Rg, dist=dict(nranks=world, rank=rank, b_lo=lo, b_hi=hi, uid=uid))
        if args.fused_gather:
            plan.set_option(OPT_FUSED_GATHER, 1)
        psi0 = x.psi[..., lo:hi].contiguous()
        order = "B (R-first) on b'-shards"
    else:
        plan = Heff(x.L, x.W1, x.W2, x.R)
        psi0 = x.psi.clone()
        order = "A (L-first)"
    stream = torch.cuda.current_stream()

    def barrier():
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up: W Lanczos steps (the Krylov workspace for the timed call is allocated
    # first, so no cudaMalloc/cudaFree falls inside the timed region)
    plan.set_option(OPT_LANCZOS_RESERVE, max(args.warmup, args.steps))
    v = psi0.clone()
    plan.lanczos_ground(v, max_iter=max(1, args.warmup))
    barrier()

    # ---- timed: K Lanczos steps (one lanczos_ground call, fixed-step mode)
    plan.set_option(OPT_PROFILE, 1)
    plan.set_option(OPT_TOTAL_LAUNCHES, 0)
    clk = Clocks(local)
    v = psi0.clone()
    barrier()
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = plan.lanczos_ground(v, max_iter=args.steps)
    e1.record(stream)
    barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    launches = plan.get_option(OPT_TOTAL_LAUNCHES)
    g1_ms, mpo_ms, g4_ms, nrec = plan.last_timings()
    plan.set_option(OPT_PROFILE, 0)
    ms_max = hdist.max_over_ranks(ms, device=dev) if sharded else ms
    value = args.steps / (ms_max / 1e3)

    # ---- e2e: heff_apply_host (pinned host psi in, host out) per step
    # every rank copies the full psi in (pinned host) and its out-shard back, per step
    e2e = None
    if args.e2e_steps > 0:
        hin = x.psi.cpu().pin_memory()
        hout = torch.empty(plan.out_shape, dtype=torch.float64).pin_memory()
        plan.apply_host(hin, hout)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.apply_host(hin, hout)
        el = time.perf_counter() - t0
        if sharded:
            el = hdist.max_over_ranks(el, device=dev)
        e2e = {"value": args.e2e_steps / el, "unit": "matvec/s", "h2d_bytes_per_step": hin.numel() * 8 * world,
               "d2h_bytes_per_step": hout.numel() * 8 * world,
               "what": "heff_apply_host on every rank: pinned-host psi -> device, H_eff.psi (its b'-shard at N>1), "
                       "device -> pinned-host out; bytes summed over ranks"}

    # ---- roofline of the dominant kernel (a GEMM step; the two GEMMs are ~50/50)
    n_mv = max(1.0, nrec)
    d = dims
    g1_flop = 2.0 * d["mL"] * d["kL"] * d["mL"] * d["d1"] * d["d2"] * d["mR"]
    g4_flop = gemm_flops - g1_flop
    if sharded:
        g1_flop /= world
        g4_flop /= world
    k1 = ("gemm_first", g1_ms, g1_flop)
    k4 = ("gemm_last", g4_ms, g4_flop)
    dom = max((k1, k4), key=lambda k: k[1])
    per_launch_ms = dom[1] / n_mv
    achieved = dom[2] / (per_launch_ms / 1e3) / 1e12 if per_launch_ms > 0 else None
    kernel_names = {"gemm_first": "gemm_dmma_tma_kernel NT (psi.R_g^T)" if sharded else "gemm_dmma_tma_kernel NN (L.psi)",
                    "gemm_last": "gemm_dmma_tma_kernel NN (L.V3)" if sharded else "gemm_dmma_tma_kernel NT (T3.R^T)"}
    traffic, traffic_src = load_ncu_traffic(dom[0] + ("_B" if sharded else "_A"))
    roofline = {"bound": "tensor", "kernel": kernel_names[dom[0]], "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS if achieved else None,
                "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "derived FP64 DMMA peak 148 SM x 128 flop/clk x 1.965 GHz = 37.2 TF/s (no FP64 entry "
                               "in MEASURED_PEAKS.json); DMMA microbenchmark 37.16 TF/s sustained",
                "per_launch_ms": per_launch_ms,
                "gemm_steps": {"gemm_first_tflops": g1_flop * n_mv / (g1_ms / 1e3) / 1e12 if g1_ms else None,
                               "gemm_last_tflops": g4_flop * n_mv / (g4_ms / 1e3) / 1e12 if g4_ms else None,
                               "gemm_both_frac": ((g1_flop + g4_flop) * n_mv / ((g1_ms + g4_ms) / 1e3) / 1e12
                                                  / FP64_PEAK_TFLOPS) if (g1_ms + g4_ms) else None,
                               "mpo_ms_per_matvec": mpo_ms / n_mv,
                               "share_of_step": {"gemm_first": g1_ms / ms, "mpo": mpo_ms / ms, "gemm_last": g4_ms / ms}}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        del plan
        torch.cuda.empty_cache()
        cpu = cpu_baseline(x.to("cpu"))

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": bench_config(args.config, dims, flops),
                "layout": {"order": order,
                           "parallelism": (f"b'-shard x{world} (" + ("gather-fused GEMM_A on NCCL symmetric-window "
                                           "peer pointers" if args.fused_gather else "NCCL all-gather") + ")")
                           if sharded else "single GPU"},
                "tflops": value * flops / 1e12, "frac_fp64_peak": value * flops / 1e12 / (FP64_PEAK_TFLOPS * world),
                "lanczos": {"energy": res.energy, "iters": res.iters},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks}
        print(json.dumps(line), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
