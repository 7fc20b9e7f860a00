"""Multi-strip (multi-GPU) paths at the BASELINE cfg5 shape and through the
library's own multi-strip engine.

The reference splits the lattice into row strips (make_strip_plan +
worker_rows, backends.cpp:20-36, 140-145; run_strips :149-219) and its
tests require every strip count to give the single-domain bits
(test_backends.cpp:118-133). The same holds here for:

* fhpg_create_multi (Engine(..., strips=n)): the library owns n strip
  engines and exchanges the halo rows itself (peer copies, overlapped with
  the interior rows);
* LocalStrips: n strip engines driven from Python with fhpg_advance_part;
* DistStrips over two processes, each with a real CUDA strip engine, the
  halo rows staged through host memory and exchanged over gloo.

Only one GPU is available to these tests, so every strip sits on cuda:0; the
cross-device copies take the same code path (cudaMemcpyPeerAsync).
cfg4/cfg5: 16384 x 16384 split into 2 and 4 strips, 20 steps, must give the
digest the reference itself produced (tests/golden/golden_long.json); the
8190- and 4094-row interior launches take the ring kernel's extra-CTA split.
"""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1208_2428_b200 as P
from paper_1208_2428_b200.strips import DistStrips, LocalStrips, strip_rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LONG = os.path.join(ROOT, "tests", "golden", "golden_long.json")


def _cfg4():
    return next(c for c in json.load(open(LONG))["configs"] if c["name"] == "cfg4")


def test_multi_engine_rejects_bad_strip_counts():
    # make_strip_plan's errors come before any device is touched
    for n in (0, 9):
        with pytest.raises(P.FhpgInvalidArgument, match="strip count"):
            P.Engine(64, 10, strips=n)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 5])
@pytest.mark.parametrize("W,H", [(2048, 70), (1024, 41), (512, 70), (100, 41)])
def test_multi_engine_equals_oracle(n, W, H, port, tables):
    for tname, fp in (("fhp3", 0.2), ("default", 0.0)):
        state, mask = port.scramble(W, H, 31 * n + W)
        e = P.Engine(W, H, strips=n, devices=[0] * n)
        assert [s[:2] for s in e.strips] == strip_rows(H, n)
        e.set_table(tables[tname])
        e.set_obstacles(mask)
        e.upload(state)
        # steps = 0 leaves the uploaded bytes untouched (backends.cpp:157)
        assert e.advance(5, fp, 3, 0) == 0
        assert (e.download() == state).all()
        sw = e.advance(5, fp, 3, 7)
        sw += e.advance(5, fp, 10, 4)  # a second call continues the step sequence
        ref, rsw = port.advance(state, tables[tname], 5, port.threshold(fp), 3, 11, mask=mask)
        out = e.download()
        assert (out == ref).all(), (W, H, n, tname)
        assert sw == rsw
        # observables summed over the strips == the whole lattice's
        whole = P.Engine(W, H)
        whole.set_table(tables[tname])
        whole.set_obstacles(mask)
        whole.upload(out)
        assert e.observables() == whole.observables()
        for k, (a, b) in enumerate(zip(e.cells(4), whole.cells(4))):
            assert (a == b).all(), k
        for a, b in zip(e.rows(), whole.rows()):
            assert (a == b).all()
        e.close()
        whole.close()


@pytest.mark.gpu
def test_multi_engine_rejects_single_strip_calls():
    e = P.Engine(1024, 20, strips=2, devices=[0, 0])
    with pytest.raises(P.FhpgInvalidArgument):
        e.set_stream(None)
    with pytest.raises(P.FhpgInvalidArgument):
        e.halo()
    with pytest.raises(P.FhpgInvalidArgument):
        e.advance_part(1, 0, 0, 0)
    e.close()


@pytest.mark.gpu
def test_multi_engine_init_equals_whole(tables, port):
    W, H = 4096, 301
    mask = port.cylinder(W, H)
    e = P.Engine(W, H, strips=4, devices=[0] * 4)
    e.set_table(tables["fhp3"])
    e.set_obstacles(mask)
    e.init(11, 0.3)
    w = P.Engine(W, H)
    w.set_table(tables["fhp3"])
    w.set_obstacles(mask)
    w.init(11, 0.3)
    assert (e.download() == w.download()).all()
    assert e.advance(11, 0.05, 0, 9) == w.advance(11, 0.05, 0, 9)
    assert (e.download() == w.download()).all()


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 4])
def test_cfg5_multi_engine_digest(n, tables, port):
    c = _cfg4()
    e = P.Engine(c["W"], c["H"], strips=n, devices=[0] * n)
    e.set_table(tables["fhp3"])
    e.init(c["seed"], c["density"])
    assert e.path == "planes"
    e.advance(c["seed"], c["force_p"], 0, 12)
    e.advance(c["seed"], c["force_p"], 12, c["steps"] - 12)
    assert port.digest(e.download()) == c["digest"]
    assert list(e.observables()) == c["obs"]
    e.close()


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 4])
def test_cfg5_local_strips_digest(n, tables, port):
    c = _cfg4()
    ls = LocalStrips(c["W"], c["H"], n)
    ls.set_table(tables["fhp3"])
    ls.init(c["seed"], c["density"])
    assert all(e.path == "planes" for e in ls.engines)
    assert ls.advance(c["seed"], c["force_p"], 0, c["steps"]) == c["swaps"]
    assert port.digest(ls.download()) == c["digest"]


def _cuda_worker(rank, world, port_num, W, H, steps, seed, fp, init, q):
    import datetime
    import sys
    import traceback
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_num))
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=180))
        sys.path.insert(0, ROOT)
        import paper_1208_2428_b200 as P
        from oracle.oracle import Port  # checker only (scrambled input)
        torch.cuda.set_device(0)
        rb, re = strip_rows(H, world)[rank]
        eng = P.Engine(W, H, rb, re, 0)
        eng.set_table(P.build_table("fhp3"))
        if init:
            eng.init(seed, 0.2)
        else:
            state, mask = Port().scramble(W, H, seed)
            eng.set_obstacles(mask[rb:re])
            eng.upload(state[rb:re])
        strips = DistStrips(eng, rank, world, staging="host")
        swaps = strips.advance(seed, P.bernoulli_threshold(fp), 0, steps)
        sizes = [b - a for a, b in strip_rows(H, world)]
        mine = torch.zeros((max(sizes), W), dtype=torch.uint8)  # gloo gathers equal sizes
        mine[: re - rb] = torch.from_numpy(eng.download())
        if rank == 0:
            parts = [torch.empty((max(sizes), W), dtype=torch.uint8) for _ in sizes]
            dist.gather(mine, parts, dst=0)
            rows = torch.cat([p[:k] for p, k in zip(parts, sizes)])
            q.put(("ok", rows.numpy(), swaps))
        else:
            dist.gather(mine, None, dst=0)
        eng.close()
        dist.destroy_process_group()
    except BaseException:
        q.put(("err", f"rank {rank}: " + traceback.format_exc(), None))
        raise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_cuda_world(world, W, H, steps, seed, fp, init):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = mp.start_processes(_cuda_worker,
                               args=(world, _free_port(), W, H, steps, seed, fp, init, q),
                               nprocs=world, join=False, start_method="spawn")
    status, got, swaps = q.get(timeout=400)
    for p in procs.processes:
        p.join(timeout=60 if status == "ok" else 5)
        if p.is_alive():
            p.kill()
    assert status == "ok", got
    return got, swaps


@pytest.mark.gpu
def test_dist_strips_cuda_engines_gloo(port, tables):
    W, H, steps, seed, fp = 2048, 131, 9, 4242, 0.3
    got, swaps = _run_cuda_world(2, W, H, steps, seed, fp, init=False)
    state, mask = port.scramble(W, H, seed)
    ref, rsw = port.advance(state, tables["fhp3"], seed, port.threshold(fp), 0, steps, mask=mask)
    assert (got == ref).all()
    assert swaps == rsw


@pytest.mark.gpu
@pytest.mark.slow
def test_dist_strips_cuda_engines_gloo_cfg4(port):
    c = _cfg4()
    got, swaps = _run_cuda_world(2, c["W"], c["H"], c["steps"], c["seed"], c["force_p"], init=True)
    assert port.digest(got) == c["digest"]
    assert swaps == c["swaps"]
