"""Regenerates tests/golden/ from the REFERENCE's own fixture generator.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports /root/reference/proj/data/gen_fixtures.py and uses its writer
functions (msh22/msh41/structured) so the committed meshes are byte-identical
to what the reference generator emits; it also records the SHA-256 of the
14,192-cell gear produced by the same recipe at n_r=16, n_t=887,
which the product's procedural gear generator must reproduce bit for bit.
Nothing here is read from /root/reference at test time.
"""
import hashlib
import importlib.util
import json
import math
import os

REF = "/root/reference/proj/data/gen_fixtures.py"
HERE = os.path.dirname(os.path.abspath(__file__))


def load_ref():
    spec = importlib.util.spec_from_file_location("gen_fixtures", REF)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def gear_text(g, n_r, n_t, teeth=12, amp=0.06, r_in=0.35, r_out=1.0):
    # exactly the recipe of gen_fixtures.py main() (lines 158-179), parametrised
    nodes = []
    for j in range(n_r + 1):
        s = j / n_r
        for i in range(n_t):
            th = 2 * math.pi * i / n_t
            r = r_in + s * (r_out + amp * math.sin(teeth * th) - r_in)
            nodes.append((r * math.cos(th), r * math.sin(th)))
    nid = lambda i, j: j * n_t + (i % n_t) + 1
    quads = []
    for j in range(n_r):
        for i in range(n_t):
            quads.append((nid(i, j), nid(i, j + 1), nid(i + 1, j + 1), nid(i + 1, j)))
    g.check_valid(nodes, quads, "gear")
    lines = [(nid(i, 0), nid(i + 1, 0)) for i in range(n_t)]
    lines += [(nid(i, n_r), nid(i + 1, n_r)) for i in range(n_t)]
    return g.msh41(nodes, quads, lines)


def main():
    g = load_ref()
    out = os.path.join(HERE, "meshes")
    os.makedirs(out, exist_ok=True)
    # Re-run the reference generator into our golden dir.
    g.OUT = out
    g.main()
    # Bundled fixtures must equal what the generator wrote (sanity).
    for name in sorted(os.listdir(out)):
        ref_file = os.path.join(os.path.dirname(REF), "meshes", name)
        if os.path.exists(ref_file):
            assert open(ref_file).read() == open(os.path.join(out, name)).read(), name
    gear576 = gear_text(g, 6, 96)
    assert gear576 == open(os.path.join(out, "gearlike_v41.msh")).read()
    gear14k = gear_text(g, 16, 887)
    info = {
        "gear_14192": {
            "n_r": 16, "n_t": 887,
            "sha256": hashlib.sha256(gear14k.encode()).hexdigest(),
            "n_bytes": len(gear14k.encode()),
            "first_lines": gear14k.splitlines()[:12],
            "last_lines": gear14k.splitlines()[-6:],
        }
    }
    # the reference's own run configs (must keep loading unchanged)
    import shutil
    cfg_out = os.path.join(HERE, "configs")
    os.makedirs(cfg_out, exist_ok=True)
    for name in sorted(os.listdir("/root/reference/proj/configs")):
        shutil.copy(os.path.join("/root/reference/proj/configs", name), os.path.join(cfg_out, name))
    with open(os.path.join(HERE, "gear_14192.json"), "w") as fh:
        json.dump(info, fh, indent=1)
    print("golden meshes and gear_14192.json written")


if __name__ == "__main__":
    main()
