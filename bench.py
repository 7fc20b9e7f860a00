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
through fhp::run_bench on the host cores, on the same 16384 x 16384 lattice,
loading the same FHP-III table from data/fhp3.fhptab with its own
read_table_file; it imports nothing from this framework.

`--gpus N` without torchrun re-executes itself under torch.distributed.run
(one process per GPU, 127.0.0.1 rendezvous); rank 0 prints the line.
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
TABLE_FILE = os.path.join(ROOT, "data", "fhp3.fhptab")  # FHPTAB01, `fhp_b200 tablegen --rules fhp3`
CPU_DIGEST_STEPS = 10   # cpu_baseline: 1 warm-up + 10 timed steps of the full lattice
MATRIX_ROWS = 256       # lanes x1 / scalar x1: a 16384 x 256 slab of the same workload


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def int_roof(table, peak_bw_gbs):
    """SURVEY 8(d)'s second roof: integer ops per site at the INT32 peak.
    Algorithmic ops = 22 (one mix64 on sm_100a) x (f_chir + f_force): the
    chirality / forcing draws the path cannot avoid; f_chir exact for i.i.d.
    density-d states (each chirality slice of the table is a permutation, so
    states stay i.i.d.), f_force = 0 at p = 0. The peak is the measured
    half-rate LOP3/SHF/IMAD lane rate (profiles/int_peaks_r01.json). The
    implementation's own ALU-pipe instructions per site (ncu, when the
    committed summary has them) give the roof this kernel actually faces."""
    d = DENSITY
    f_chir = 0.0
    for st in range(128):
        if table[st] != table[256 + st]:
            k = bin(st).count("1")
            f_chir += d ** k * (1 - d) ** (7 - k)
    f_force = d * (1 - d) if FORCE_P > 0 else 0.0
    ops = 22.0 * (f_chir + f_force)
    peak = None
    try:
        with open(os.path.join(ROOT, "profiles", "int_peaks_r01.json")) as f:
            peak = float(json.load(f)["kernels"]["lop3"]["lane_ops_per_s"])
    except Exception:
        peak = 148 * 64 * 1.965e9  # half-rate INT pipe at the max SM clock
    out = {"ops_per_site": ops, "f_chir": f_chir, "f_force": f_force,
           "peak_lane_ops_per_s": peak, "roof_gsups": peak / ops / 1e9,
           "hbm_roof_gsups": peak_bw_gbs / BYTES_PER_SITE}
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_step_kernel.json")) as f:
            alu = json.load(f).get("alu_inst_per_site")
        if alu:
            out["impl_alu_inst_per_site"] = alu
            out["impl_alu_roof_gsups"] = peak / alu / 1e9
    except Exception:
        pass
    out["bound"] = "hbm" if out["hbm_roof_gsups"] <= out["roof_gsups"] else "int"
    return out


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


def ref_lib():
    from oracle.oracle import Ref  # checker / baseline only (never the measured product)
    return Ref()


def cpu_run(ref, W, H, steps, warmup, backend="strips", threads=None):
    """fhp::run_bench(cfg) of the reference library on the host cores, the
    FHP-III table read by the reference itself from the FHPTAB01 file."""
    return ref.bench_file(W, H, steps, warmup, DENSITY, FORCE_P, SEED, table_file=TABLE_FILE,
                          backend=backend, threads=threads, repeats=1)


def cpu_matrix(ref):
    """BASELINE.md's other CPU arms, lanes x1 and scalar x1, on a bounded slab."""
    out = {}
    for backend in ("lanes", "scalar"):
        r = cpu_run(ref, W_LAT, MATRIX_ROWS, 3, 1, backend=backend, threads=1)
        out[f"{backend}x1"] = {"value": r["mups"] / 1000.0, "unit": "GSUPS", "cores": 1,
                               "sample": f"{W_LAT}x{MATRIX_ROWS} slab, 1 warmup + 3 timed steps"}
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = ref_lib()
    threads = os.cpu_count()
    W, H = W_LAT, H_PER_GPU
    res = cpu_run(ref, W, H, args.steps, args.warmup, threads=threads)
    gsups = res["mups"] / 1000.0
    world = args.gpus
    sample = (f"{W}x{H} lattice (cfg4, one GPU's share of cfg5 at N={world}), fhp::run_bench strips "
              f"x {threads} threads, {args.warmup} warmup + {args.steps} timed steps, FHP-III read "
              f"from data/fhp3.fhptab by the reference's read_table_file")
    line = {"metric": METRIC, "value": gsups, "unit": "GSUPS", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["wall_seconds"] * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "cfg4/cfg5: FHP-III 16384x16384 per GPU, x-periodic, walls "
                                   "rows 0/H-1, d=0.2, seed 4, p=0",
                       "W": W, "H": H, "table": "FHP-III (data/fhp3.fhptab)",
                       "same_config": world == 1,
                       "digest": f"{res['digest']:#018x}",
                       "digest_after_steps": args.warmup + args.steps},
            "cpu_baseline": {"value": gsups, "unit": "GSUPS", "cores": threads,
                             "kind": "reference", "sample": sample},
            "cpu_matrix": cpu_matrix(ref),
            "e2e": {"value": gsups, "unit": "GSUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(args):
    """`--gpus N` outside torchrun: re-run this script under
    torch.distributed.run with N local ranks (rank 0 prints)."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="print the launch plan (ranks, strips) and exit without a GPU")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    from paper_1208_2428_b200.strips import strip_rows
    H = H_PER_GPU * world
    rb, re = strip_rows(H, world)[rank]
    if args.dry_run:
        print(json.dumps({"dry_run": True, "rank": rank, "world": world, "local_rank": local,
                          "W": W_LAT, "H": H, "rows": [rb, re]}), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    import paper_1208_2428_b200 as P
    from paper_1208_2428_b200.strips import DistStrips

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    table = P.build_table("fhp3")
    eng = P.Engine(W_LAT, H, rb, re, local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    eng.set_table(table)
    eng.init(SEED, DENSITY)
    thr = P.bernoulli_threshold(FORCE_P)
    strips = DistStrips(eng, rank, world)  # puts the engine on `stream` (NCCL's ordering stream)

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
    gpu_launches = eng.step_launches - launches0  # step kernels + column keys
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        g = torch.tensor([gpu_launches], device="cuda", dtype=torch.int64)
        dist.all_reduce(g)
        gpu_launches = int(g.item())
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
                         "l2": "inputs larger than L2 (2 x 272 MB state buffers per GPU)",
                         "kernel": {"planes": "bit-plane ring kernel (step_ring_kernel)",
                                    "bytes": "byte streaming kernel (step_fast_kernel)",
                                    "generic": "generic"}[eng.path]},
              "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                           "frac": achieved / peak, "traffic": traffic,
                           "bytes_per_site": BYTES_PER_SITE, "peak_source": peak_src,
                           "int": int_roof(table, peak),
                           "timing": "CUDA events on the engine stream around the K-step loop, "
                                     "per-step average (one step kernel per step at N=1)"},
              "gpu_launches": gpu_launches,
              "clocks": clk.summary()}
    if world == 1:
        # Parity stamp: the state after warmup + K steps (compare with the
        # reference arm's digest at the same step count).
        result["config"]["digest"] = f"{P.state_digest(eng.download()):#018x}"
        result["config"]["digest_after_steps"] = args.warmup + args.steps
    eng.close()
    if not args.no_e2e:
        e2e = e2e_measure(P, table, args, world, rank, rb, re, barrier)
        if rank == 0:
            result["e2e"] = e2e
    barrier()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(P, table, local)
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


def cpu_baseline(P, table, device):
    """The reference library on the host cores (all threads) on the full
    16384^2 lattice for 1 + CPU_DIGEST_STEPS steps, and the same steps on the
    GPU: the two digests must agree."""
    import torch
    ref = ref_lib()
    threads = os.cpu_count()
    res = cpu_run(ref, W_LAT, H_PER_GPU, CPU_DIGEST_STEPS, 1, threads=threads)
    e = P.Engine(W_LAT, H_PER_GPU, 0, H_PER_GPU, device)
    e.set_table(table)
    e.init(SEED, DENSITY)
    e.advance(SEED, FORCE_P, 0, 1 + CPU_DIGEST_STEPS)
    gpu_digest = P.state_digest(e.download())
    e.close()
    torch.cuda.synchronize()
    return {"value": res["mups"] / 1000.0, "unit": "GSUPS", "cores": threads, "kind": "reference",
            "sample": f"{W_LAT}x{H_PER_GPU} (the full per-GPU lattice), fhp::run_bench of "
                      f"oracle/_ref (reference proj/core built from source), strips x {threads} "
                      f"threads, 1 warmup + {CPU_DIGEST_STEPS} timed steps",
            "digest": f"{res['digest']:#018x}", "gpu_digest": f"{gpu_digest:#018x}",
            "digest_match": res["digest"] == gpu_digest}


def e2e_measure(P, table, args, world, rank, rb, re, barrier):
    """fhp::advance through the C ABI on host buffers (the Backend::Cuda shim
    of INTEGRATION.md with a cached engine): H2D of state + obstacle mask
    from pinned memory, K steps (halo exchange included at N > 1), D2H of the
    state and the swap count, all inside the timed region; wall clock around
    synchronous calls, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_1208_2428_b200.strips import DistStrips
    W, rows = W_LAT, re - rb
    src = P.Engine(W, world * H_PER_GPU, rb, re, torch.cuda.current_device())
    src.set_table(table)
    src.init(SEED, DENSITY)
    host = torch.empty((rows, W), dtype=torch.uint8, pin_memory=True).numpy()
    src.download(host)
    mask = torch.empty((rows, W), dtype=torch.uint8, pin_memory=True).numpy()
    np.right_shift(host, 7, out=mask)
    src.close()
    e = P.Engine(W, world * H_PER_GPU, rb, re, torch.cuda.current_device())
    e.set_table(table)
    strips = DistStrips(e, rank, world)
    thr = P.bernoulli_threshold(FORCE_P)
    # warm-up of the path
    e.set_obstacles(mask)
    e.upload(host)
    strips.advance(SEED, thr, 0, 3)
    torch.cuda.synchronize()
    out = torch.empty((rows, W), dtype=torch.uint8, pin_memory=True).numpy()
    barrier()
    t0 = time.perf_counter()
    e.set_obstacles(mask)
    e.upload(host)
    strips.advance(SEED, thr, args.warmup, args.steps)
    e.download(out)
    t1 = time.perf_counter()
    e.close()
    secs = t1 - t0
    if world > 1:
        t = torch.tensor([secs], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs = float(t.item())
    h2d = 2 * W * rows  # state + obstacle mask (per rank)
    d2h = W * rows + 8  # state + swap count
    return {"value": W * world * H_PER_GPU * args.steps / secs / 1e9, "unit": "GSUPS",
            "h2d_bytes_per_step": world * h2d / args.steps,
            "d2h_bytes_per_step": world * d2h / args.steps,
            "call": f"fhpg_set_obstacles+fhpg_upload+fhpg_advance({args.steps} steps)+"
                    "fhpg_download on pinned host buffers"
                    + (" per rank, halo exchange over NCCL" if world > 1 else ""),
            "seconds": secs}


if __name__ == "__main__":
    sys.exit(main())
