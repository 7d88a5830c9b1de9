"""Structural comparison of result JSON with a floating-point tolerance."""
import math


def assert_close(a, b, rel=1e-6, path="$"):
    if isinstance(a, float) or isinstance(b, float):
        assert isinstance(a, (int, float)) and isinstance(b, (int, float)), f"{path}: {a!r} vs {b!r}"
        if a == b:
            return
        assert math.isclose(a, b, rel_tol=rel, abs_tol=1e-12), f"{path}: {a!r} vs {b!r}"
        return
    assert type(a) == type(b), f"{path}: type {type(a).__name__} vs {type(b).__name__} ({a!r} vs {b!r})"
    if isinstance(a, dict):
        assert sorted(a) == sorted(b), f"{path}: keys {sorted(a)} vs {sorted(b)}"
        for k in a:
            assert_close(a[k], b[k], rel, f"{path}.{k}")
    elif isinstance(a, list):
        assert len(a) == len(b), f"{path}: len {len(a)} vs {len(b)}"
        for i, (x, y) in enumerate(zip(a, b)):
            assert_close(x, y, rel, f"{path}[{i}]")
    else:
        assert a == b, f"{path}: {a!r} vs {b!r}"


def assert_flags_match(got, exp, rel=1e-9):
    """flag_ranks lists [(rank, name, frac, threshold)]: identical, except that a
    flag decided by a near-tie (|frac - threshold| <= rel) may differ — the
    waterline's fractions are count/total, within 1e-6 of the reference's
    line-order sums, so an exact tie can land on either side."""
    g = {(f[0], f[1]): f for f in got}
    e = {(f[0], f[1]): f for f in exp}
    for k in set(g) ^ set(e):
        f = g.get(k) or e.get(k)
        frac, thr = f[2], f[3]
        assert abs(frac - thr) <= rel * max(abs(frac), abs(thr), 1e-300), f"flag {k} differs: {f}"
    for k in set(g) & set(e):
        assert math.isclose(g[k][2], e[k][2], rel_tol=1e-6) and math.isclose(g[k][3], e[k][3], rel_tol=1e-6)
