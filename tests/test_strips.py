"""Row-strip decomposition (the multi-GPU path).

* strip_rows mirrors make_strip_plan + worker_rows (backends.cpp:20-36,
  140-145; test_backends.cpp:118-133 cases).
* CPU, world_size 2 and 3 over gloo: DistStrips' halo exchange protocol with
  an oracle-backed strip engine gives the single-domain digest exactly.
* GPU: LocalStrips (several real strip engines on one device, halo copies
  between them) gives the single-engine bits for 1..5 strips.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1208_2428_b200.strips import DistStrips, strip_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_strip_rows_matches_reference_plan():
    # make_strip_plan(10, 3) = [(1,4), (4,7), (7,9)] plus the wall rows
    assert strip_rows(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert strip_rows(5, 1) == [(0, 5)]
    for H in (3, 8, 33, 99):
        for n in range(1, H - 1):
            rows = strip_rows(H, n)
            assert rows[0][0] == 0 and rows[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 2
    with pytest.raises(ValueError):
        strip_rows(10, 9)
    with pytest.raises(ValueError):
        strip_rows(10, 0)


class OracleStrip:
    """CPU stand-in for one strip engine: same halo/advance interface, the
    step computed by the oracle (test infrastructure)."""

    def __init__(self, port, W, H, rb, re, state, mask, table):
        self.port, self.W, self.H, self.rb, self.re = port, W, H, rb, re
        self.buf = np.zeros((re - rb + 2, W), np.uint8)
        self.buf[1:-1] = state[rb:re]
        self.mask = np.ascontiguousarray(mask[rb:re])
        self.table = table
        self.sw = 0

    def halo_tensors(self):
        t = torch.from_numpy(self.buf)
        n = self.re - self.rb
        return t[1], t[n], t[0], t[n + 1]

    def advance_async(self, seed, thr, first, count):
        for s in range(first, first + count):
            out, sw = self.port.step_strip(self.H, self.rb, self.buf, self.mask, self.table, seed,
                                           thr, s)
            self.buf[1:-1] = out
            self.sw += sw

    def advance_part(self, seed, thr, step, part):
        # The oracle has no row split: the whole step runs at part 1, after
        # the halos have arrived (part 0 must not need them).
        if part == 1:
            self.advance_async(seed, thr, step, 1)

    def swaps(self, reset=False):
        v = self.sw
        if reset:
            self.sw = 0
        return v


def _worker(rank, world, port_num, W, H, steps, seed, fp, table_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_num))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    import json
    from oracle.oracle import Port
    port = Port()
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    table = np.frombuffer(bytes.fromhex(g["tables"][table_name]), np.uint8).copy()
    state, mask = port.scramble(W, H, seed)
    rb, re = strip_rows(H, world)[rank]
    eng = OracleStrip(port, W, H, rb, re, state, mask, table)
    strips = DistStrips(eng, rank, world, halo_tensors=eng.halo_tensors)
    swaps = strips.advance(seed, port.threshold(fp), 3, steps)
    rows = [None] * world
    dist.all_gather_object(rows, eng.buf[1:-1].copy())
    if rank == 0:
        q.put((np.concatenate(rows, axis=0), swaps))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,W,H,table_name", [(2, 48, 21, "fhp3"), (3, 33, 17, "default")])
def test_dist_strips_gloo_equals_single_domain(world, W, H, table_name, port, tables):
    steps, seed, fp = 9, 4242, 0.3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), W, H, steps, seed, fp, table_name, q),
                       nprocs=world, join=True, start_method="spawn")
    got, swaps = q.get(timeout=60)
    state, mask = port.scramble(W, H, seed)
    ref, rsw = port.advance(state, tables[table_name], seed, port.threshold(fp), 3, steps,
                            mask=mask)
    assert (got == ref).all()
    assert swaps == rsw


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_local_strips_gpu_equal_single_engine(n, port, tables):
    import paper_1208_2428_b200 as P
    from paper_1208_2428_b200.strips import LocalStrips
    for (W, H) in ((512, 70), (100, 41)):
        state, mask = port.scramble(W, H, 77 + n)
        ls = LocalStrips(W, H, n)
        ls.set_table(tables["fhp3"])
        ls.set_obstacles(mask)
        ls.upload(state)
        sw = ls.advance(5, 0.2, 10, 12)
        out = ls.download()
        ref, rsw = port.advance(state, tables["fhp3"], 5, port.threshold(0.2), 10, 12, mask=mask)
        assert (out == ref).all(), (W, H, n)
        assert sw == rsw
        # device init of the strips == whole-lattice device init
        ls2 = LocalStrips(W, H, n)
        ls2.set_table(tables["fhp3"])
        ls2.init(9, 0.3)
        whole = P.Engine(W, H)
        whole.set_table(tables["fhp3"])
        whole.init(9, 0.3)
        assert (ls2.download() == whole.download()).all()
        # observables of strips sum to the whole lattice's
        m = sum(e.observables()[0] for e in ls2.engines)
        assert m == whole.observables()[0]
        cells = [e.cells(4) for e in ls2.engines]
        wc = whole.cells(4)
        for k in range(4):
            assert (sum(c[k] for c in cells) == wc[k]).all()


@pytest.mark.parametrize("n", [2, 4])
def test_bench_spawns_its_own_ranks(n):
    """`python bench.py --gpus N` outside torchrun re-executes itself under
    torch.distributed.run with N ranks (the driver's SCALE invocation); each
    rank takes its row strip of the weak-scaled N x 16384-row lattice."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                        "--dry-run"], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(s) for s in r.stdout.splitlines() if s.startswith("{")]
    assert sorted(d["rank"] for d in lines) == list(range(n))
    assert all(d["world"] == n and d["H"] == 16384 * n for d in lines)
    rows = sorted(tuple(d["rows"]) for d in lines)
    assert rows == strip_rows(16384 * n, n)
