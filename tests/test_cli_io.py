"""Formats and tool layer on CPU: the dataset CSV reader
and writer follow io.cpp:70-152 (header forms, blank lines, error messages),
the model JSON round-trips in the "gradkrig-model" v1 layout of
model_io.cpp:12-153 and rejects what load_model rejects, the CLI maps errors
onto the exit codes of proj/tools/common.hpp:14-18 / common.cpp:86-100, and
the host RNG pieces the tools use (uniform_real_distribution over
seeded_rng, the precond-study sample_dataset) equal the oracle's. No GPU
work is done here."""
import json

import numpy as np
import pytest

import oracle as O
from paper_1810_12283_b200 import cli
from paper_1810_12283_b200 import io as gio


def _write(p, text):
    p.write_text(text)
    return str(p)


def test_read_dataset_csv_header_forms(tmp_path):
    path = _write(tmp_path / "d.csv", "X2, y ,x1,G1,g2\r\n1.5,2,0.5,3,4\n\n  \n-1e-3,0,7,8,9\n")
    d = gio.read_dataset_csv(path)
    assert d.X.tolist() == [[0.5, 1.5], [7.0, -1e-3]]
    assert d.y.tolist() == [2.0, 0.0]
    assert d.G.tolist() == [[3.0, 4.0], [8.0, 9.0]]
    # value-only file and an input-only file for prediction (y zero-filled)
    d = gio.read_dataset_csv(_write(tmp_path / "v.csv", "x1,y\n1,2\n"))
    assert not d.has_gradients
    d = gio.read_dataset_csv(_write(tmp_path / "t.csv", "x1,x2\n1,2\n"), require_y=False)
    assert d.y.tolist() == [0.0]


@pytest.mark.parametrize("text, msg", [
    ("", "empty file"),
    ("x1,z\n", "unrecognized header column 'z'"),
    ("x0,y\n", "bad header column 'x0'"),
    ("x1\n1\n", "missing 'y' column"),
    ("y\n1\n", "missing x columns"),
    ("x1,x2,y,g1\n1,2,3,4\n", "gradient columns must match the input dimension"),
    ("x1,y\n1,2,3\n", "row 2 has 3 cells, expected 2"),
    ("x1,y\n1,\n", "malformed number '' at row 2, column 2"),
    ("x1,y\n1,2x\n", "malformed number '2x' at row 2, column 2"),
])
def test_read_dataset_csv_errors(tmp_path, text, msg):
    with pytest.raises(RuntimeError, match=msg):
        gio.read_dataset_csv(_write(tmp_path / "bad.csv", text))


def test_missing_file_message(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open"):
        gio.read_dataset_csv(str(tmp_path / "nope.csv"))


def test_dataset_csv_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    d = gio.Dataset(rng.standard_normal((7, 3)), rng.standard_normal(7), rng.standard_normal((7, 3)) * 1e-300)
    path = str(tmp_path / "rt.csv")
    gio.write_dataset_csv(path, d)
    assert open(path).readline().strip() == "x1,x2,x3,y,g1,g2,g3"
    e = gio.read_dataset_csv(path)
    assert np.array_equal(e.X, d.X) and np.array_equal(e.y, d.y) and np.array_equal(e.G, d.G)


def test_observation_validation():
    d = gio.Dataset(np.array([[0.0], [np.nan]]), np.zeros(2))
    with pytest.raises(ValueError, match="non-finite"):
        d.to_observations(0.1, 0.1)
    with pytest.raises(ValueError, match="empty"):
        gio.Dataset(np.zeros((0, 1)), np.zeros(0)).to_observations(0.1, 0.1)


def test_model_json_round_trip_and_layout(tmp_path):
    m = gio.ModelFile(lengthscale=0.123456789012345, outputscale=2.5, noise_value=1e-3, noise_gradient=2e-3,
                      mean=-0.75, backend="dski",
                      config=gio.SolverConfig(backend="dski", grid_ratio=0.25, max_grid_nodes=64, cg_tol=1e-6),
                      grid={"dims": [10, 12], "origin": [-0.1, -0.2], "spacing": [0.1, 0.1]},
                      projection=np.arange(6.0).reshape(3, 2), data_path="train.csv", with_gradients=False)
    path = str(tmp_path / "m.json")
    gio.save_model(path, m)
    j = json.load(open(path))
    assert j["format"] == "gradkrig-model" and j["version"] == 1
    assert j["kernel"] == {"family": "se", "lengthscale": 0.123456789012345, "outputscale": 2.5}
    assert j["noise"] == {"value": 1e-3, "gradient": 2e-3} and j["mean"] == {"type": "constant", "value": -0.75}
    assert set(j["solver"]) == {"grid_ratio", "max_grid_nodes", "dskip_rank", "cg_tol", "cg_maxit", "precond",
                                "precond_rank", "slq_probes", "slq_steps", "seed"}
    assert list(j) == sorted(j)  # nlohmann objects are ordered maps
    r = gio.load_model(path)
    assert (r.lengthscale, r.outputscale, r.noise_value, r.noise_gradient, r.mean) == (
        m.lengthscale, m.outputscale, m.noise_value, m.noise_gradient, m.mean)
    assert r.config.grid_ratio == 0.25 and r.config.max_grid_nodes == 64 and r.config.cg_tol == 1e-6
    assert r.config.backend == "dski" and r.grid == m.grid and np.array_equal(r.projection, m.projection)
    assert r.data_path == "train.csv" and r.with_gradients is False


@pytest.mark.parametrize("doc, msg", [
    ("{", "is not valid JSON"),
    ('{"format": "other"}', "is not a gradkrig model file"),
    ('{"format": "gradkrig-model", "version": 2}', "unsupported model file version 2"),
])
def test_model_load_errors(tmp_path, doc, msg):
    with pytest.raises(RuntimeError, match=msg):
        gio.load_model(_write(tmp_path / "m.json", doc))


def test_model_load_defaults_and_aliases(tmp_path):
    doc = {"format": "gradkrig-model", "kernel": {"family": "se", "lengthscale": 0.5, "outputscale": 1.0},
           "noise": {"value": 0.1, "gradient": 0.2}, "mean": {"type": "constant", "value": 0.0},
           "backend": "ski", "data": {"path": "x.csv"}}
    m = gio.load_model(_write(tmp_path / "m.json", json.dumps(doc)))
    assert m.backend == "dski" and m.config.cg_maxit == 1000 and m.config.precond and m.with_gradients
    doc["backend"] = "gpu"
    with pytest.raises(ValueError, match="unknown backend 'gpu'"):
        gio.load_model(_write(tmp_path / "m2.json", json.dumps(doc)))
    doc["backend"] = "dski"
    doc["grid"] = {"dims": [1, 2], "origin": [0.0], "spacing": [1.0, 1.0]}
    with pytest.raises(RuntimeError, match="grid descriptor is inconsistent"):
        gio.load_model(_write(tmp_path / "m3.json", json.dumps(doc)))


def test_cli_exit_codes_without_device_work(tmp_path):
    data = _write(tmp_path / "d.csv", "x1,x2,y\n0.1,0.2,1\n0.3,0.4,2\n")
    assert cli.main(["fit", "--data", str(tmp_path / "missing.csv")]) == cli.EXIT_DATA
    assert cli.main(["fit", "--data", _write(tmp_path / "bad.csv", "x1,y\n1,oops\n")]) == cli.EXIT_DATA
    assert cli.main(["fit", "--data", data, "--backend", "gpu"]) == cli.EXIT_CONFIG  # not a backend
    assert cli.main(["fit", "--data", data, "--precond", "maybe"]) == cli.EXIT_CONFIG  # parse error
    assert cli.main(["fit"]) == cli.EXIT_CONFIG  # --data is required
    # "is not a gradkrig model file" matches none of common.cpp:92-98's data
    # patterns: the reference classifies it as a solver failure (3)
    assert cli.main(["predict", "--model", _write(tmp_path / "m.json", "{}"), "--test", data]) == cli.EXIT_SOLVER
    assert cli.main(["predict", "--model", str(tmp_path / "none.json"), "--test", data]) == cli.EXIT_DATA
    assert cli.main(["precond-study", "--function", "branin"]) == cli.EXIT_CONFIG


def test_classify_exception_matches_reference_rules():
    import paper_1810_12283_b200 as gk
    assert cli.classify_exception(gk.OutOfGridError("point 3 outside the grid", 3)) == cli.EXIT_DATA
    assert cli.classify_exception(ValueError("bad")) == cli.EXIT_CONFIG
    assert cli.classify_exception(RuntimeError("CG did not converge: ...")) == cli.EXIT_SOLVER
    assert cli.classify_exception(RuntimeError("all fit restarts failed: [x]")) == cli.EXIT_SOLVER
    assert cli.classify_exception(RuntimeError("f.csv: row 3 has 2 cells")) == cli.EXIT_DATA
    assert cli.classify_exception(RuntimeError("something else")) == cli.EXIT_SOLVER


def test_uniform_vector_is_libstdcxx_uniform_real_distribution():
    """uniform_real_distribution<double>(a, b) over mt19937_64: one raw draw u
    per value, canonical = u / 2^64 (generate_canonical), value =
    canonical·(b − a) + a — checked against the oracle's raw engine."""
    import paper_1810_12283_b200 as gk
    seed, stream = 3, 33
    got = gk.uniform_vector(50, seed, stream, -0.7, 0.7)
    s = O.mix_seed(seed, stream)
    for i in range(50):
        c = float(O.mt19937_64_nth(s, i + 1)) / 2.0 ** 64
        assert got[i] == c * 1.4 + -0.7


@pytest.mark.parametrize("name, noise", [("franke", (0.0, 0.0)), ("friedman", (0.1, 0.05))])
def test_sample_test_function_bit_identical_to_oracle(name, noise):
    import paper_1810_12283_b200 as gk
    a = gk.sample_test_function(name, 257, 4, noise)
    b = O.sample_test_function(name, 257, 4, noise)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    with pytest.raises(ValueError, match="unknown test function"):
        gk.sample_test_function("branin", 10)


def test_benchmark_points_follow_seeded_rng_row_order():
    X = cli.bench_points(5, 3, 2)
    u = O.mix_seed(2, 5)
    flat = [float(O.mt19937_64_nth(u, i + 1)) / 2.0 ** 64 for i in range(15)]
    assert X.flatten(order="C").tolist() == flat


def test_spline_constants_for_domain():
    """SplineConstants::for_domain (kernels.cpp:42-90): a = −1.5·D, the first
    PSD b on the canonical lattice, doubled; the b before it is not PSD."""
    import paper_1810_12283_b200 as gk
    for D, dim in ((2.0, 2), (3.5, 3), (1.2, 1), (4.0, 5)):
        a, b, even = gk.spline_constants_for_domain(D, dim)
        assert a == -1.5 * D and even == (dim % 2 == 0)
        mult = b / 2 / D ** 3
        assert mult in [0.25 * 2 ** j for j in range(13)]
        axes = min(dim, 3)
        side = D / np.sqrt(axes)
        idx = np.arange(5 ** axes)
        P = np.column_stack([side * ((idx // 5 ** ax) % 5) / 4 for ax in range(axes)])
        R = np.sqrt(((P[:, None] - P[None]) ** 2).sum(-1))
        with np.errstate(divide="ignore", invalid="ignore"):
            rad = np.where(R > 0, R * R * np.log(np.where(R > 0, R, 1.0)), 0.0) if even else R ** 3
        ev = np.linalg.eigvalsh(rad + a * R * R + b / 2)
        assert ev.min() >= -1e-10 * ev.max()
        if mult > 0.25:
            ev = np.linalg.eigvalsh(rad + a * R * R + b / 4)
            assert ev.min() < -1e-10 * ev.max()
    with pytest.raises(ValueError):
        gk.spline_constants_for_domain(0.0, 2)
