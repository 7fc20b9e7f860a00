"""FHP lattice-gas throughput on B200 (BASELINE.json metric: site updates/s, GSUPS).

Workload (BASELINE configs[3]/[4]): FHP-III on a
16384 x 16384 lattice per GPU (x-periodic, wall rows 0 and H-1 as in the
reference), reference init_lattice with seed 4, density 0.2, no forcing.
N GPUs: weak scaling, one 16384-row strip per rank of a 16384 x 16384N
lattice, halo rows exchanged over NVLink every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0). `value` = whole-job GSUPS with the state
resident in HBM, device-timed with CUDA events on the engine's stream, max
over ranks; `e2e` = the same metric through the reference-facing C-ABI call
(fhpg_upload + fhpg_advance + fhpg_download on pinned host buffers, the
`case Backend::Cuda` shim of fhp::advance) with the copies inside the timed
region. The reference arm times the reference library itself
(oracle/_ref/libfhpref.so = /root/reference/proj/core compiled from source)
through fhp::run_bench on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_LAT = 16384
H_PER_GPU = 16384
SEED = 4
DENSITY = 0.2
FORCE_P = 0.0
BYTES_PER_SITE = 1.875  # 7 state bits read + 7 written + 1 obstacle bit
METRIC = "FHP site updates/s (GSUPS) at 1/2/4/8 B200; fraction of HBM roofline"
CPU_SAMPLE_ROWS = 2048  # reference CPU sample: 16384 x 2048 slab of the same workload


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per step-kernel launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_step_kernel.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if d.get("W") == W_LAT and d.get("rows") == H_PER_GPU:
            return d.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


class ClockSampler:
    """NVML SM clock + throttle reasons, sampled in a thread during timing."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    _NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
              0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
              0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
              0x100: "display_clock_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_reference(W, H, steps, warmup, table, threads=None):
    """fhp::run_bench(cfg) of the reference library on the host cores."""
    from oracle.oracle import Ref  # checker / baseline only
    ref = Ref()
    res = ref.bench(W, H, steps, warmup, DENSITY, FORCE_P, SEED, table=table, backend="strips",
                    threads=threads or os.cpu_count(), repeats=1)
    return res


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import paper_1208_2428_b200 as P
    table = P.build_table("fhp3")
    threads = os.cpu_count()
    res = cpu_reference(W_LAT, CPU_SAMPLE_ROWS, args.steps, args.warmup, table, threads)
    gsups = res["mups"] / 1000.0
    sample = (f"{W_LAT}x{CPU_SAMPLE_ROWS} slab of the cfg4 workload (FHP-III, d=0.2, seed 4, "
              f"p=0), fhp::run_bench strips x {threads} threads, {args.warmup} warmup + "
              f"{args.steps} timed steps")
    line = {"metric": METRIC, "value": gsups, "unit": "GSUPS", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["wall_seconds"] * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "cfg4: FHP-III 16384x16384/GPU, x-periodic, walls rows 0/H-1, "
                                   "d=0.2, seed 4, p=0 (CPU: bounded row slab)",
                       "W": W_LAT, "H": CPU_SAMPLE_ROWS, "table": "FHP-III",
                       "digest": f"{res['digest']:#018x}"},
            "cpu_baseline": {"value": gsups, "unit": "GSUPS", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": gsups, "unit": "GSUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_1208_2428_b200 as P
    from paper_1208_2428_b200.strips import DistStrips, strip_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    H = H_PER_GPU * world
    rb, re = strip_rows(H, world)[rank]
    table = P.build_table("fhp3")
    eng = P.Engine(W_LAT, H, rb, re, local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    eng.set_table(table)
    eng.init(SEED, DENSITY)
    thr = P.bernoulli_threshold(FORCE_P)
    strips = DistStrips(eng, rank, world)

    def barrier():
        if world > 1:
            dist.barrier()

    # Warm-up (untimed).
    strips.advance_async(SEED, thr, 0, args.warmup)
    torch.cuda.synchronize()

    launches0 = eng.step_launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        strips.advance_async(SEED, thr, args.warmup, args.steps)
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = start.elapsed_time(end)
    step_launches = eng.step_launches - launches0
    # column-key launches: one per advance call
    calls = args.steps if world > 1 else 1
    gpu_launches = step_launches + calls
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    sites = W_LAT * H  # all ranks
    value = sites * args.steps / (ms * 1e-3) / 1e9
    ms_per_step = ms / args.steps

    # Roofline of the step kernel: algorithmic bytes per launch / launch time.
    peak, peak_src = peaks()
    own_sites = W_LAT * (re - rb)
    achieved = own_sites * BYTES_PER_SITE / (ms_per_step * 1e-3) / 1e9
    traffic = ncu_traffic()

    result = {"metric": METRIC, "value": value, "unit": "GSUPS", "n_gpus": world,
              "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
              "data": "synthetic (reference init_lattice: seed 4, density 0.2)",
              "config": {"workload": "cfg4/cfg5: FHP-III 16384x16384 per GPU, x-periodic, walls "
                                     "rows 0/H-1, d=0.2, seed 4, p=0; row strips across GPUs",
                         "W": W_LAT, "H": H, "rows_per_gpu": H_PER_GPU, "table": "FHP-III",
                         "parallelism": f"row-strips x{world}" if world > 1 else "single",
                         "l2": "inputs larger than L2 (2 x 268 MB state buffers per GPU)",
                         "kernel": {"planes": "bit-plane ring kernel (step_ring_kernel)",
                                    "bytes": "byte streaming kernel (step_fast_kernel)",
                                    "generic": "generic"}[eng.path]},
              "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                           "frac": achieved / peak, "traffic": traffic,
                           "bytes_per_site": BYTES_PER_SITE, "peak_source": peak_src,
                           "timing": "CUDA events on the engine stream around the K-step loop, "
                                     "per-step average (one step kernel per step)"},
              "gpu_launches": gpu_launches,
              "clocks": clk.summary()}

    # Parity stamp of the timed run: digest after warmup+K steps vs nothing (informational).
    if rank == 0 and world == 1 and not args.no_e2e:
        result["e2e"] = e2e_measure(P, table, args, thr)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count()
        res = cpu_reference(W_LAT, CPU_SAMPLE_ROWS, 10, 1, table, threads)
        result["cpu_baseline"] = {
            "value": res["mups"] / 1000.0, "unit": "GSUPS", "cores": threads, "kind": "reference",
            "sample": f"{W_LAT}x{CPU_SAMPLE_ROWS} slab of the same workload, fhp::run_bench "
                      f"(oracle/_ref = reference proj/core built from source), strips x {threads} "
                      f"threads, 1 warmup + 10 timed steps"}
    eng.close()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_measure(P, table, args, thr):
    """fhp::advance through the C ABI on host buffers (the Backend::Cuda shim):
    H2D of state + mask, K steps, D2H of the state, all inside the timed
    region (wall clock around synchronous calls; pinned host memory)."""
    import torch
    W, H = W_LAT, H_PER_GPU
    src = P.Engine(W, H)
    src.set_table(table)
    src.init(SEED, DENSITY)
    host = torch.empty((H, W), dtype=torch.uint8, pin_memory=True).numpy()
    src.download(host)
    mask = torch.empty((H, W), dtype=torch.uint8, pin_memory=True).numpy()
    np.right_shift(host, 7, out=mask)
    src.close()
    e = P.Engine(W, H)
    e.set_table(table)
    # warm-up of the path
    e.set_obstacles(mask)
    e.upload(host)
    e.advance(SEED, FORCE_P, 0, 3)
    torch.cuda.synchronize()
    out = torch.empty((H, W), dtype=torch.uint8, pin_memory=True).numpy()
    t0 = time.perf_counter()
    e.set_obstacles(mask)
    e.upload(host)
    e.advance(SEED, FORCE_P, args.warmup, args.steps)
    e.download(out)
    t1 = time.perf_counter()
    e.close()
    secs = t1 - t0
    h2d = 2 * W * H  # state + obstacle mask
    d2h = W * H + 8  # state + swap count
    return {"value": W * H * args.steps / secs / 1e9, "unit": "GSUPS",
            "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
            "call": f"fhpg_set_obstacles+fhpg_upload+fhpg_advance({args.steps} steps)+fhpg_download "
                    "on pinned host buffers", "seconds": secs}


if __name__ == "__main__":
    sys.exit(main())
