"""Helpers that restate the reference tests' own fixtures (test-side only)."""
import numpy as np

MASK = (1 << 64) - 1


class SplitMix:
    """core.hpp:119-154 in Python (for synthetic_eval, test_losses.cpp:19-40)."""

    def __init__(self, seed):
        self.s = seed & MASK
        self.next()
        self.next()

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self, lo=0.0, hi=1.0):
        u = float(self.next() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u if (lo, hi) != (0.0, 1.0) else u

    def integer(self, n):
        return int(self.uniform() * float(n))


def synthetic_eval(n, seed, with_eps=False, n_scalars=0):
    """tests/test_losses.cpp:19-40 — interleaved per-point draws."""
    r = SplitMix(seed)
    u, ux, uy = np.zeros(n), np.zeros(n), np.zeros(n)
    for i in range(n):
        u[i] = r.uniform(-1.0, 1.0)
        ux[i] = r.uniform(-2.0, 2.0)
        uy[i] = r.uniform(-2.0, 2.0)
    eps = None
    if with_eps:
        eps = np.array([r.uniform(0.1, 1.5) for _ in range(n)])
    scal = [r.uniform(0.2, 2.0) for _ in range(n_scalars)]
    return u, ux, uy, eps, scal


def read_msh(path):
    """Minimal gmsh 2.2/4.1 ASCII reader used to feed fixture meshes to the
    oracle (quads only; CCW normalisation as mesh_io.hpp:234-242)."""
    lines = [l.strip() for l in open(path).read().splitlines()]
    ver = lines[lines.index("$MeshFormat") + 1].split()[0]
    tags, xy, quads = [], [], []
    i = lines.index("$Nodes") + 1
    if ver == "2.2":
        n = int(lines[i]); i += 1
        for k in range(n):
            t, x, y, _ = lines[i + k].split()
            tags.append(int(t)); xy.append((float(x), float(y)))
        i = lines.index("$Elements") + 1
        n = int(lines[i]); i += 1
        for k in range(n):
            f = list(map(int, lines[i + k].split()))
            if f[1] == 3:
                quads.append(f[3 + f[2]:])
    else:
        nb = int(lines[i].split()[0]); i += 1
        for _ in range(nb):
            cnt = int(lines[i].split()[3]); i += 1
            tt = [int(lines[i + k]) for k in range(cnt)]; i += cnt
            for k in range(cnt):
                x, y, _ = lines[i + k].split(); xy.append((float(x), float(y)))
            tags += tt; i += cnt
        i = lines.index("$Elements") + 1
        nb = int(lines[i].split()[0]); i += 1
        for _ in range(nb):
            h = lines[i].split(); typ, cnt = int(h[2]), int(h[3]); i += 1
            for k in range(cnt):
                f = list(map(int, lines[i + k].split()))
                if typ == 3:
                    quads.append(f[1:])
            i += cnt
    idx = {t: j for j, t in enumerate(tags)}
    nodes = np.array(xy)
    cells = np.array([[idx[t] for t in q] for q in quads], dtype=np.int32)
    for c in cells:
        p = nodes[c]
        a = 0.5 * sum(p[k, 0] * p[(k + 1) % 4, 1] - p[(k + 1) % 4, 0] * p[k, 1] for k in range(4))
        if a < 0:
            c[1], c[3] = c[3], c[1]
    return nodes, cells
