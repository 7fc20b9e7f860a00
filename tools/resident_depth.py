"""cfg1 throughput vs the resident kernel's halo depth (lib/ab/res<d>.so)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); import bench_configs as b, json; "
        "print(json.dumps(b.timed(1024, 1024, 'fhp1', 0.0, 1000, 1, 0.2, clear_rest=True)))") % (ROOT, os.path.join(ROOT, "tools"))
for d in sys.argv[1:]:
    env = dict(os.environ, FHPG_LIB=os.path.join(ROOT, "paper_1208_2428_b200", "lib", "ab", f"res{d}.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    print(json.dumps({"depth": int(d), "result": line}))
