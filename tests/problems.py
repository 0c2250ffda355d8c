"""Test problem generators (test infrastructure).

``random_problem`` restates testutil::random_problem (tests/helpers.hpp:29-109)
on top of the oracle's NormalGen so the same seeds give the same problems as
the reference's own unit tests.
"""
import json

from oracle.oracle import CONFIGS, NormalGen


def random_problem(seed, max_l=4, max_mult=64, max_x_segments=3, max_y_segments=2,
                   max_instructions=4, max_dense_entries=2_000_000):
    attempt = 0
    while True:
        gen = NormalGen((seed * 7919 + attempt * 104729 + 13) % (1 << 64))
        attempt += 1
        x = []
        nx = 1 + gen.below(max_x_segments)
        for _ in range(nx):
            mult = 1 + gen.below(max_mult)
            l = gen.below(max_l + 1)
            par = "e" if (gen.bits() & 1) else "o"
            x.append((mult, l, par))
        y = []
        ny = 1 + gen.below(max_y_segments)
        for _ in range(ny):
            l = gen.below(max_l + 1)
            par = "e" if (gen.bits() & 1) else "o"
            y.append((1, l, par))
        z = []
        ins = []
        ni = 1 + gen.below(max_instructions)
        for _ in range(ni):
            xs = 1 + gen.below(nx)
            ys = 1 + gen.below(ny)
            bx, by = x[xs - 1], y[ys - 1]
            lo, hi = abs(bx[1] - by[1]), min(bx[1] + by[1], max_l)
            if lo > hi:
                continue
            l3 = lo + gen.below(hi - lo + 1)
            p3 = "o" if ((bx[2] == "o") != (by[2] == "o")) else "e"
            kind = "B" if (gen.bits() & 1) else "C"
            mz = bx[0] if kind == "B" else 1 + gen.below(max_mult)
            zs = 0
            if (gen.bits() & 3) == 0:
                for k, bz in enumerate(z):
                    if bz[1] == l3 and bz[2] == p3 and bz[0] == mz:
                        zs = k + 1
                        break
            if zs == 0:
                z.append((mz, l3, p3))
                zs = len(z)
            ins.append([xs, ys, zs, kind])
        if not ins:
            continue
        fmt = lambda ir: " + ".join(f"{m}x{l}{p}" for m, l, p in ir)
        # validate() of the generated problem always passes by construction
        # (parity and triangle respected); keep the dense-size cap.
        dim_y = sum(2 * l + 1 for _, l, _ in y)
        dim_x = sum(m * (2 * l + 1) for m, l, _ in x)
        zpre = 0
        for xs, ys, zs, kind in ins:
            bz, bx = z[zs - 1], x[xs - 1]
            zpre += (bz[0] if kind == "B" else bx[0]) * (2 * bz[1] + 1)
        if dim_y * dim_x * zpre > max_dense_entries:
            continue
        return json.dumps({"x": fmt(x), "y": fmt(y), "z": fmt(z), "instructions": ins})


def config(name):
    return json.dumps(CONFIGS[name])
