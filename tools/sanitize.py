"""Small runs of every step kernel for compute-sanitizer (memcheck,
racecheck, initcheck, synccheck): the bit-plane ring kernel (W >= 2048, with
and without forcing; FHP-III, DEFAULT and FHP-I circuits), at the bench width
W = 16384 with the extra-CTA band switch (H = 1100) and with re-keying every
few rows (fhpg_debug_key_span), the per-warp bit-plane kernel (W = 1024 x
odd), the shared-memory-resident kernel, the byte fast path and the generic
path, plus a 3-strip engine on one device (fhpg_create_multi: interior /
boundary-row launches, halo peer copies) and the observables and the
asynchronous coarse-grain pipeline on each.
    python tools/sanitize.py [quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
cases = [  # W, H, force_p, rule, path, key span cap, strips
    (2048, 64, 0.2, "fhp3", "streaming", None, None),
    (4096, 131, 0.0, "fhp3", "streaming", None, None),
    (4096, 70, 0.3, "default", "streaming", None, None),
    (4096, 70, 0.0, "fhp1", "streaming", None, None),
    (16384, 1100, 0.0, "default", "streaming", 50, None),
    (4096, 70, 0.3, "fhp3", "streaming", 3, None),
    (16384, 1100, 0.0, "fhp3", "streaming", None, None),
    (16384, 1100, 0.01, "fhp3", "streaming", 100, None),
    (16384, 200, 0.0, "fhp3", "streaming", None, 3),
    (3072, 64, 0.2, "fhp3", "streaming", 5, None),
    (1024, 64, 0.2, "fhp3", "auto", None, None),
    (1024, 40, 0.0, "fhp1", "auto", None, None),
    (528, 40, 0.0, "fhp3", "auto", None, None),
    (100, 23, 0.5, "fhp3", "auto", None, None),
]
if quick:
    cases = [c for c in cases if c[0] * c[1] <= 4096 * 131]
for W, H, fp, rule, path, cap, strips in cases:
    e = P.Engine(W, H, strips=strips, devices=[0] * strips) if strips else P.Engine(W, H)
    if not strips:
        e.select_path(path)
    e.set_table(P.build_table(rule))
    if cap is not None:
        e.debug_key_span(cap)
    e.init(3, 0.3)
    e.advance(3, fp, 0, 3)
    e.observables()
    e.cells(4)
    e.cells_async(32)
    e.advance(3, fp, 3, 1)
    e.cells_wait()
    e.rows()
    e.download()
    print(W, H, rule, e.path, "cap", cap, "strips", strips, flush=True)
    e.close()
print("sanitize run ok")
