"""Data formats of the gradkrig tools: the dataset CSV
(io.cpp:70-152), the plain CSV report writer (io.cpp:243-259) and the
versioned model JSON "gradkrig-model" v1 (model_io.cpp:12-153). Host-side
file handling only; the models these files describe run on the device.

Errors follow the reference's messages (the CLI maps them onto exit codes,
proj/tools/common.cpp:86-100): RuntimeError("cannot open '...'"),
RuntimeError("<path>: malformed number '...' at row R, column C"), ...;
ValueError for the std::invalid_argument cases."""
from __future__ import annotations

import dataclasses
import json
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

BACKEND_NAMES = {"exact": "exact", "dense": "exact", "dski": "dski", "ski": "dski", "dskip": "dskip",
                 "skip": "dskip"}


def backend_from_string(name: str) -> str:
    """backend_from_string (gp.cpp:26-31), aliases included."""
    try:
        return BACKEND_NAMES[name]
    except KeyError:
        raise ValueError(f"unknown backend '{name}'") from None


def format_number(v: float) -> str:
    """%.17g (io.cpp:44-48): round-trips every double."""
    return "%.17g" % v


def _trim(s: str) -> str:
    return s.strip(" \t\r\n")


def _split_csv_line(line: str):
    """io.cpp:21-27: split on ',' and trim each cell; an empty line has no
    cells, a trailing ',' gives one trailing empty cell (str.split agrees
    with std::getline + the re-added cell in every other case)."""
    return [] if line == "" else [_trim(c) for c in line.split(",")]


def _parse_number(token: str, row: int, col: int, path: str) -> float:
    """io.cpp:29-42: std::stod must consume the whole (trimmed) token."""
    try:
        if "_" in token:  # Python-only digit separators
            raise ValueError
        return float(token)
    except ValueError:
        raise RuntimeError(f"{path}: malformed number '{token}' at row {row + 1}, column {col + 1}") from None


@dataclass
class Dataset:
    """Dataset (io.hpp:13-25): X n×d, y n, G n×d or None (value-only)."""
    X: np.ndarray
    y: np.ndarray
    G: Optional[np.ndarray] = None

    @property
    def has_gradients(self) -> bool:
        return self.G is not None and self.G.size > 0

    def dim(self) -> int:
        return int(self.X.shape[1])

    def points(self) -> int:
        return int(self.X.shape[0])

    def to_observations(self, noise_value: float, noise_gradient: float):
        """Dataset::to_observations (io.cpp:51-60) + ObservationSet::validate
        (observations.hpp:37-44). Returns (X, y, dY or None)."""
        X, y = self.X, self.y
        dY = self.G if self.has_gradients else None
        if X.shape[0] < 1:
            raise ValueError("observation set is empty")
        if y.shape[0] != X.shape[0]:
            raise ValueError("y has wrong length")
        if dY is not None and dY.shape != X.shape:
            raise ValueError("gradient block must be n x d (all-or-none per set)")
        if not (np.all(np.isfinite(X)) and np.all(np.isfinite(y)) and (dY is None or np.all(np.isfinite(dY)))):
            raise ValueError("observations contain non-finite entries")
        return X, y, dY


def read_dataset_csv(path: str, require_y: bool = True) -> Dataset:
    """read_dataset_csv (io.cpp:70-134): header x1..xD, y, optional g1..gD
    (any order, case-insensitive), then numeric rows; blank lines skipped."""
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise RuntimeError(f"cannot open '{path}'") from None
    with f:
        lines = f.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise RuntimeError(f"{path}: empty file")
    header = _split_csv_line(lines[0])
    dim = gdim = 0
    ycol = -1
    xcols = [-1] * len(header)
    gcols = [-1] * len(header)
    for c, h0 in enumerate(header):
        h = h0.lower()
        if h == "y":
            ycol = c
        elif len(h) > 1 and h[0] in "xg":
            idx = _atoi(h[1:])
            if idx <= 0:
                raise RuntimeError(f"{path}: bad header column '{h0}'")
            if h[0] == "x":
                xcols[c] = idx - 1
                dim = max(dim, idx)
            else:
                gcols[c] = idx - 1
                gdim = max(gdim, idx)
        else:
            raise RuntimeError(f"{path}: unrecognized header column '{h0}'")
    if ycol < 0 and require_y:
        raise RuntimeError(f"{path}: missing 'y' column")
    if dim == 0:
        raise RuntimeError(f"{path}: missing x columns")
    if gdim != 0 and gdim != dim:
        raise RuntimeError(f"{path}: gradient columns must match the input dimension")
    rows = []
    for line in lines[1:]:
        if _trim(line) == "":
            continue
        cells = _split_csv_line(line)
        r = len(rows)
        if len(cells) != len(header):
            raise RuntimeError(f"{path}: row {r + 2} has {len(cells)} cells, expected {len(header)}")
        rows.append([_parse_number(cell, r + 1, c, path) for c, cell in enumerate(cells)])
    n = len(rows)
    X = np.zeros((n, dim))
    y = np.zeros(n)
    G = np.zeros((n, dim)) if gdim > 0 else None
    for i, vals in enumerate(rows):
        for c, v in enumerate(vals):
            if c == ycol:
                y[i] = v
            elif xcols[c] >= 0:
                X[i, xcols[c]] = v
            elif gcols[c] >= 0:
                G[i, gcols[c]] = v
    return Dataset(np.asfortranarray(X), y, np.asfortranarray(G) if G is not None else None)


def _atoi(s: str) -> int:
    """std::atoi: leading whitespace, optional sign, digits; 0 if none."""
    s = s.lstrip()
    k = 0
    if k < len(s) and s[k] in "+-":
        k += 1
    j = k
    while j < len(s) and s[j].isdigit():
        j += 1
    return int(s[:j]) if j > k else 0


def write_dataset_csv(path: str, data: Dataset) -> None:
    """write_dataset_csv (io.cpp:136-152)."""
    d = data.dim()
    header = [f"x{j + 1}" for j in range(d)] + ["y"] + ([f"g{j + 1}" for j in range(d)] if data.has_gradients
                                                      else [])
    rows = []
    for i in range(data.points()):
        row = list(data.X[i]) + [data.y[i]]
        if data.has_gradients:
            row += list(data.G[i])
        rows.append(row)
    write_csv(path, header, rows)


def write_csv(path: str, header, rows) -> None:
    """write_csv (io.cpp:243-259): header row, then %.17g cells."""
    try:
        f = open(path, "w", newline="")
    except OSError:
        raise RuntimeError(f"cannot write '{path}'") from None
    with f:
        f.write(",".join(header) + "\n")
        for row in rows:
            f.write(",".join(format_number(float(v)) for v in row) + "\n")


# ------------------------------------------------------------------ model JSON
@dataclass
class SolverConfig:
    """The GpConfig fields the model file echoes (model_io.cpp:32-43; GpConfig gp.hpp:23-48)."""
    backend: str = "exact"
    grid_ratio: float = 0.2
    max_grid_nodes: int = 128
    dskip_rank: int = 100
    cg_tol: float = 1e-4
    cg_maxit: int = 1000
    precond: bool = True
    precond_rank: int = 100
    slq_probes: int = 10
    slq_steps: int = 50
    gradient_probes: int = 8
    seed: int = 0


@dataclass
class ModelFile:
    """ModelFile (model_io.hpp:16-29)."""
    version: int = 1
    family: str = "se"
    lengthscale: float = 1.0
    outputscale: float = 1.0
    spline_a: float = -1.5
    spline_b: float = 1.0
    spline_even: bool = False
    noise_value: float = 1e-2
    noise_gradient: float = 1e-2
    mean: float = 0.0
    backend: str = "exact"
    config: SolverConfig = field(default_factory=SolverConfig)
    grid: Optional[dict] = None  # {"dims", "origin", "spacing"}
    projection: Optional[np.ndarray] = None  # D×d active-subspace matrix
    data_path: str = ""
    with_gradients: bool = True


def _num(v):
    """JSON numbers as nlohmann writes them: integers stay integers, doubles
    round-trip (non-finite values are written as null)."""
    if isinstance(v, (bool, np.bool_)):
        return bool(v)
    if isinstance(v, (int, np.integer)):
        return int(v)
    v = float(v)
    return v if math.isfinite(v) else None


def save_model(path: str, m: ModelFile) -> None:
    """save_model (model_io.cpp:12-73). Keys are written sorted (nlohmann::json
    objects are ordered maps), indent 2."""
    k = {"family": m.family, "lengthscale": _num(m.lengthscale), "outputscale": _num(m.outputscale)}
    if m.family == "spline":
        k.update(spline_a=_num(m.spline_a), spline_b=_num(m.spline_b), spline_even=bool(m.spline_even))
    c = m.config
    j = {
        "format": "gradkrig-model",
        "version": int(m.version),
        "kernel": k,
        "noise": {"value": _num(m.noise_value), "gradient": _num(m.noise_gradient)},
        "mean": {"type": "constant", "value": _num(m.mean)},
        "backend": m.backend,
        "solver": {"grid_ratio": _num(c.grid_ratio), "max_grid_nodes": int(c.max_grid_nodes),
                   "dskip_rank": int(c.dskip_rank), "cg_tol": _num(c.cg_tol), "cg_maxit": int(c.cg_maxit),
                   "precond": bool(c.precond), "precond_rank": int(c.precond_rank),
                   "slq_probes": int(c.slq_probes), "slq_steps": int(c.slq_steps), "seed": int(c.seed)},
        "data": {"path": m.data_path, "with_gradients": bool(m.with_gradients)},
    }
    if m.grid is not None:
        j["grid"] = {"dims": [int(v) for v in m.grid["dims"]], "origin": [_num(v) for v in m.grid["origin"]],
                     "spacing": [_num(v) for v in m.grid["spacing"]]}
    if m.projection is not None:
        j["projection"] = [[_num(v) for v in row] for row in np.asarray(m.projection)]
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot write model file '{path}'") from None
    with f:
        f.write(json.dumps(j, indent=2, sort_keys=True) + "\n")


def load_model(path: str) -> ModelFile:
    """load_model (model_io.cpp:75-153): format/version checks, optional
    solver block (absent keys keep the GpConfig defaults), grid and projection
    consistency checks."""
    try:
        f = open(path, "r")
    except OSError:
        raise RuntimeError(f"cannot open model file '{path}'") from None
    with f:
        try:
            j = json.load(f)
        except json.JSONDecodeError as e:
            raise RuntimeError(f"model file '{path}' is not valid JSON: {e}") from None
    if not isinstance(j, dict) or j.get("format", "") != "gradkrig-model":
        raise RuntimeError(f"'{path}' is not a gradkrig model file")
    m = ModelFile()
    m.version = int(j.get("version", 1))
    if m.version != 1:
        raise RuntimeError(f"unsupported model file version {m.version}")
    try:
        k = j["kernel"]
        m.family = k["family"]
        if m.family not in ("se", "spline"):
            raise ValueError(f"unknown kernel family '{m.family}'")
        if m.family == "spline":
            m.spline_a, m.spline_b = float(k["spline_a"]), float(k["spline_b"])
            m.spline_even = bool(k.get("spline_even", False))
        m.lengthscale, m.outputscale = float(k["lengthscale"]), float(k["outputscale"])
        m.noise_value = float(j["noise"]["value"])
        m.noise_gradient = float(j["noise"]["gradient"])
        m.mean = float(j["mean"]["value"])
        m.backend = backend_from_string(j["backend"])
        c = SolverConfig()
        if "solver" in j:
            s = j["solver"]
            c = dataclasses.replace(
                c, grid_ratio=float(s.get("grid_ratio", c.grid_ratio)),
                max_grid_nodes=int(s.get("max_grid_nodes", c.max_grid_nodes)),
                dskip_rank=int(s.get("dskip_rank", c.dskip_rank)), cg_tol=float(s.get("cg_tol", c.cg_tol)),
                cg_maxit=int(s.get("cg_maxit", c.cg_maxit)), precond=bool(s.get("precond", True)),
                precond_rank=int(s.get("precond_rank", c.precond_rank)),
                slq_probes=int(s.get("slq_probes", c.slq_probes)), slq_steps=int(s.get("slq_steps", c.slq_steps)),
                seed=int(s.get("seed", c.seed)))
        c.backend = m.backend
        m.config = c
        if "grid" in j:
            g = j["grid"]
            dims, origin, spacing = list(g["dims"]), list(g["origin"]), list(g["spacing"])
            if not (len(dims) == len(origin) == len(spacing)):
                raise RuntimeError("model grid descriptor is inconsistent")
            m.grid = {"dims": [int(v) for v in dims], "origin": [float(v) for v in origin],
                      "spacing": [float(v) for v in spacing]}
        if "projection" in j:
            rows = j["projection"]
            if rows:
                if any(len(r) != len(rows[0]) for r in rows):
                    raise RuntimeError("model projection is ragged")
                m.projection = np.array(rows, dtype=np.float64)
        m.data_path = str(j["data"]["path"])
        m.with_gradients = bool(j["data"].get("with_gradients", True))
    except (KeyError, TypeError) as e:
        raise RuntimeError(f"model file '{path}' is missing a field: {e}") from None
    return m
