"""Measurement helpers with the reference's semantics (pkg/src/atamul/bench.py:57-88)
plus the seeded input generators of the five BASELINE configs."""
from __future__ import annotations

import numpy as np

from .errors import InvalidMeasurementError
from .matrix import DenseMatrix


def effective_gflops(m: int, n: int, seconds: float, r: int = 1) -> float:
    """r * m * n^2 / (seconds * 1e9) (bench.py:57-65)."""
    if seconds <= 0:
        raise InvalidMeasurementError(f"invalid measurement: {seconds} s")
    if r not in (1, 2):
        raise ValueError("r must be 1 or 2")
    return r * m * n * n / (seconds * 1e9)


def gen_matrix(m: int, n: int, seed: int, dist: str = "uniform", dtype=np.float64) -> DenseMatrix:
    """Deterministic random matrix (bench.py:68-74); dist="normal" is the
    BASELINE extension used by configs c2 and c5 (draw f64, then cast)."""
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        a = rng.uniform(-1.0, 1.0, (m, n))
    elif dist == "normal":
        a = rng.standard_normal((m, n))
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    return DenseMatrix(a.astype(dtype, copy=False))


def check_tolerance(a) -> float:
    """1e-9*m*max|A|^2 (f64) or 1e-4*m*max|A|^2 (f32) (bench.py:85-88)."""
    a = np.asarray(a)
    scale = float(np.abs(a).max()) if a.size else 1.0
    unit = 1e-9 if a.dtype == np.float64 else 1e-4
    return unit * a.shape[0] * max(scale, 1e-30) ** 2


# BASELINE.json configs
CONFIGS = {
    "c1": dict(m=1024, n=1024, seed=0, dist="uniform", dtype="f64", threshold=64 * 64),
    "c2": dict(m=6001, n=4097, seed=1, dist="normal", dtype="f64", threshold=256 * 256),
    "c3": dict(m=16384, n=16384, seed=2, dist="uniform", dtype="f64", threshold="auto"),
    "c4": dict(m=65536, n=32768, seed=3, dist="uniform", dtype="f64", threshold="auto"),
    "c5": dict(m=1048576, n=2048, seed=4, dist="normal", dtype="f32", threshold="auto"),
}


def config_matrix(name: str, rows: int | None = None) -> np.ndarray:
    """Seeded input of a config; `rows` draws only the first rows (same
    stream prefix, used for bounded CPU samples)."""
    cfg = CONFIGS[name]
    m = cfg["m"] if rows is None else rows
    dt = np.float64 if cfg["dtype"] == "f64" else np.float32
    return gen_matrix(m, cfg["n"], cfg["seed"], cfg["dist"], dt).a


def bench_plan_params(name: str, rows: int, device, base=None, autotune: bool | None = None):
    """(auto_params, precision) of the plan ``bench.py`` times on config
    `name` for a shard of `rows` rows -- shared with the full-size parity
    tests so they check exactly the benchmarked plan.  fp64 auto configs use
    ``base`` (default AutoParams()); c3, whose BASELINE cutoff is
    "auto-tuned", measures its rates and leaf width on `device`
    (autotune.tune) unless autotune=False.  c5 computes in single-pass TF32."""
    cfg = CONFIGS[name]
    f64 = cfg["dtype"] == "f64"
    precision = "fp32" if f64 else "tf32"
    if cfg["threshold"] != "auto":
        return None, precision
    from . import auto_plan
    params = base if base is not None else auto_plan.AutoParams()
    if autotune is None:
        autotune = name == "c3"
    if autotune and f64:
        from . import autotune as at
        params = at.tune(rows, cfg["n"], device, base=params)
    return params, precision
