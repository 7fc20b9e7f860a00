"""CPU check of the bit-sliced collision circuits of the bit-plane kernel
(csrc/fhpg_planes_rules.cuh): tools/planes_rules_check.cpp evaluates them on
the host (the same source the kernel compiles) for all 256 states x both
chiralities and compares with the 512-entry tables, including the exact
chirality-dependence mask that drives the lazy RNG walk."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_planes_circuits_match_tables(tmp_path):
    exe = tmp_path / "planes_rules_check"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(ROOT, "paper_1208_2428_b200", "csrc"),
                    os.path.join(ROOT, "tools", "planes_rules_check.cpp"),
                    os.path.join(ROOT, "paper_1208_2428_b200", "csrc", "fhpg_tables.cpp"),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "fhp3: ok (48 dep states)" in out.stdout
    assert "default: ok (3 dep states)" in out.stdout
    assert "fhp1: ok (3 dep states)" in out.stdout
    assert "chir_bit: ok" in out.stdout
    assert "col_key_terms: ok" in out.stdout
