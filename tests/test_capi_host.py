"""CPU-side checks of the product library (no GPU compute): the C-ABI shared
library loads and exports every symbol include/gk_capi.h declares; the host
pieces (Grid::cover, RNG streams, seeded datasets) agree with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1810_12283_b200 as gk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "gk_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(gk.LIB_PATH)
    names = declared_symbols()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python mirror binds all of them
    assert set(names) <= set(gk.EXPORTED_SYMBOLS), set(names) - set(gk.EXPORTED_SYMBOLS)


def test_library_is_sm100a_build():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gk.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_rng_streams_match_oracle():
    assert gk.mix_seed(0, 50003) == O.mix_seed(0, 50003)
    assert np.array_equal(gk.rademacher_vector(500, 3, 1001), O.rademacher_vector(500, 3, 1001))
    assert np.array_equal(gk.gaussian_vector(500, 3, 1001), O.gaussian_vector(500, 3, 1001))


@pytest.mark.parametrize("max_nodes", [12, 40, 128])
def test_grid_cover_matches_oracle(max_nodes):
    X = np.random.default_rng(4).uniform(-1, 2, (77, 3))
    a = gk.Grid.cover(X, 0.07, 3, max_nodes)
    b = O.Grid.cover(X, 0.07, 3, max_nodes)
    assert list(a.dims) == list(b.dims)
    assert np.array_equal(a.origin, b.origin) and np.array_equal(a.spacing, b.spacing)


def test_grid_cover_errors():
    with pytest.raises(ValueError):
        gk.Grid.cover(np.zeros((0, 2)), 0.1)
    with pytest.raises(ValueError):
        gk.Grid.cover(np.zeros((3, 2)), 0.0)


@pytest.mark.parametrize("cfg,n,d", [(1, 2000, 2), (2, 10000, 2), (3, 25001, 3), (5, 10000, 6)])
def test_datasets_are_seeded_and_shaped(cfg, n, d):
    X, y, dY = gk.make_dataset(cfg, 0)
    assert X.shape == (n, d) and y.shape == (n,) and dY.shape == (n, d)
    X2, y2, dY2 = gk.make_dataset(cfg, 0)
    assert np.array_equal(X, X2) and np.array_equal(y, y2) and np.array_equal(dY, dY2)
    assert np.all(np.isfinite(y)) and np.all(np.isfinite(dY))


def test_dataset_c1_analytic_gradients():
    X, y, dY = gk.make_dataset(1, 0)
    a, b = X[:, 0], X[:, 1]
    assert np.allclose(y, np.sin(6 * a) * np.cos(4 * b) + 0.5 * a * b, rtol=0, atol=1e-14)
    assert np.allclose(dY[:, 0], 6 * np.cos(6 * a) * np.cos(4 * b) + 0.5 * b, atol=1e-13)


def test_dataset_c3_normals_are_unit_and_outward():
    X, y, dY = gk.make_dataset(3, 0)
    nrm = np.linalg.norm(dY[:-1], axis=1)
    assert np.allclose(nrm, 1.0, atol=1e-12)
    assert np.all(np.sum(dY[:-1] * X[:-1], axis=1) > 0)  # star-shaped: outward
    assert y[-1] == -1.0 and np.all(X[-1] == 0.0)


def test_errors_map_to_reference_exception_types():
    # no GPU needed: argument validation happens before any device work
    with pytest.raises(ValueError):
        gk.KernelSpec(-1.0, 1.0)
    with pytest.raises(ValueError):
        gk.make_dataset(9)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_oracle_datasets_bit_identical_to_product(cfg):
    # the reference arm of bench.py and the oracle-side fixtures generate their
    # inputs with the oracle library only; both sides must see the same workload
    Xa, ya, dYa = gk.make_dataset(cfg, 0)
    Xb, yb, dYb = O.make_dataset(cfg, 0)
    assert np.array_equal(Xa, Xb) and np.array_equal(ya, yb) and np.array_equal(dYa, dYb)
    assert np.array_equal(gk.stacked_targets(ya, dYa, ya.mean()), O.stacked_targets(yb, dYb, yb.mean()))


def test_bench_reference_arm_loads_only_the_oracle():
    """bench.py --impl reference must run the reference algorithm without the
    product library: its inputs come from the oracle's own generators."""
    import subprocess
    import sys
    code = ("import sys, types; sys.argv=['bench.py']; import bench; "
            "a=types.SimpleNamespace(steps=1, warmup=0, gpus=1); line=bench.run_reference(a); "
            "maps=open('/proc/self/maps').read(); "
            "assert 'libgk_b200' not in maps, 'product library loaded'; "
            "assert 'libgk_oracle' in maps; assert 'paper_1810_12283_b200' not in sys.modules; "
            "print(line['value'] > 0)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("True")
