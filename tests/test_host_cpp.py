"""The C++ host layer (namespace fhp_b200) and the fhp_b200 CLI.

Mirrors the reference's doctest suites and test_cli.cpp: the C++ driver
tests/cpp/test_host_api.cpp checks the API against the C oracle; the CLI is
driven end to end for its subcommands and exit codes (fhp_main.cpp:163-183).
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TEST_BIN = os.path.join(ROOT, "tests", "cpp", "test_host_api")
CLI = os.path.join(ROOT, "paper_1208_2428_b200", "lib", "fhp_b200")


@pytest.fixture(scope="module", autouse=True)
def built():
    if not (os.path.exists(TEST_BIN) and os.path.exists(CLI)):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1208_2428_b200", "host")],
                       check=True, capture_output=True)


def run(*args, **kw):
    return subprocess.run(list(args), capture_output=True, text=True, timeout=600, **kw)


def test_cpp_api_host_side():
    r = run(TEST_BIN, "cpu")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_api_device_side():
    r = run(TEST_BIN, "gpu")
    assert r.returncode == 0, r.stdout + r.stderr


def test_cli_tablegen_and_validate(tmp_path, tables):
    for rules in ("default", "fhp1", "fhp3"):
        out = tmp_path / f"{rules}.tab"
        r = run(CLI, "tablegen", str(out), "--rules", rules)
        assert r.returncode == 0, r.stderr
        data = out.read_bytes()
        assert len(data) == 520 and data[:8] == b"FHPTAB01"
        assert data[8:] == tables[rules].tobytes()
        v = run(CLI, "validate", str(out))
        assert v.returncode == 0 and "valid: 512 entries, 0 violations" in v.stdout
    bad = bytearray((tmp_path / "default.tab").read_bytes())
    bad[9] = 0
    (tmp_path / "bad.tab").write_bytes(bytes(bad))
    v = run(CLI, "validate", str(tmp_path / "bad.tab"))
    assert v.returncode == 1 and "violation" in v.stdout


def test_cli_exit_codes(tmp_path):
    assert run(CLI).returncode == 2                                   # no subcommand
    assert run(CLI, "frobnicate").returncode == 2                     # unknown subcommand
    assert run(CLI, "run", "--width", "0").returncode == 2            # invalid_argument
    assert run(CLI, "run", "--bogus", "1").returncode == 2
    assert run(CLI, "run", "--width", "abc").returncode == 2
    assert run(CLI, "validate", str(tmp_path / "missing.tab")).returncode == 3  # runtime_error


def test_cli_cylinder_geometry(tmp_path, port):
    out = tmp_path / "cyl.txt"
    r = run(CLI, "geometry", str(out), "--width", "256", "--height", "128", "--cylinder")
    assert r.returncode == 0, r.stderr
    rows = out.read_text().split()
    m = port.cylinder(256, 128)
    got = np.array([[c == "#" for c in row] for row in rows], np.uint8)
    assert (got == m).all()


@pytest.mark.gpu
def test_cli_run_matches_reference_digest(tmp_path, golden):
    # 48x33, d=0.35, p=0.01, seed 5, 60 steps -> 0xf088af706ca84065
    r = run(CLI, "run", "--width", "48", "--height", "33", "--steps", "60", "--density", "0.35",
            "--force-p", "0.01", "--seed", "5", "--dump-every", "20",
            "--out-prefix", str(tmp_path / "o"))
    assert r.returncode == 0, r.stderr
    assert "digest 0xf088af706ca84065" in r.stdout
    assert "forcing_swaps 180" in r.stdout
    for step in (20, 40, 60):
        flow = (tmp_path / f"o_step{step}_flow.csv").read_text().splitlines()
        assert flow[0] == "cell_x,cell_y,rho,ux,uy" and len(flow) == 1 + 12 * 8
        prof = (tmp_path / f"o_step{step}_profile.csv").read_text().splitlines()
        assert prof[0] == "row,mean_ux,sample_count" and len(prof) == 1 + 31
        pgm = (tmp_path / f"o_step{step}_density.pgm").read_bytes()
        hdr = b"P5\n12 8\n255\n"
        assert pgm.startswith(hdr) and len(pgm) == len(hdr) + 96


@pytest.mark.gpu
def test_cli_bench(tmp_path):
    r = run(CLI, "bench", "--width", "4096", "--height", "1024", "--steps", "50", "--warmup", "5",
            "--repeats", "2", "--rules", "fhp3")
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 2 and '"backend":"cuda"' in lines[0]


@pytest.mark.gpu
def test_cli_checkpoint_resume(tmp_path):
    # f4: run 60 steps straight == run 25 (checkpoint every 10) + resume to 60.
    common = ["--width", "48", "--height", "33", "--density", "0.35", "--force-p", "0.01",
              "--seed", "5"]
    r = run(CLI, "run", "--steps", "60", *common)
    assert r.returncode == 0 and "digest 0xf088af706ca84065" in r.stdout, r.stderr
    ck = tmp_path / "ck.bin"
    a = run(CLI, "run", "--steps", "25", *common, "--checkpoint-file", str(ck),
            "--checkpoint-every", "10")
    assert a.returncode == 0, a.stderr
    from paper_1208_2428_b200 import checkpoint as K
    c = K.load(str(ck))
    assert (c.width, c.height, c.next_step, c.seed, c.force_p) == (48, 33, 25, 5, 0.01)
    b = run(CLI, "run", "--steps", "60", "--resume", str(ck))
    assert b.returncode == 0, b.stderr
    assert "digest 0xf088af706ca84065" in b.stdout and "forcing_swaps 180" in b.stdout
    # mismatching resume requests are invalid_argument (exit 2); a corrupt file exit 3
    assert run(CLI, "run", "--steps", "20", "--resume", str(ck)).returncode == 2
    raw = bytearray(ck.read_bytes())
    raw[-1] ^= 1
    (tmp_path / "bad.bin").write_bytes(bytes(raw))
    assert run(CLI, "run", "--steps", "60", "--resume", str(tmp_path / "bad.bin")).returncode == 3
