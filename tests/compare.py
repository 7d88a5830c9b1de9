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
