"""DSS model container and the dss-v1 weights format.

Mirrors the model half of the reference's pkg/src/ddmgnn/dss.py: the
dataclasses Mlp / IterationWeights / DssModel (:54-81), param_count (:84-86),
the canonical parameter order (:93-99), Xavier init (:102-127) and the dss-v1
reader/writer (:530-571).  Inference itself runs on the GPU (csrc/gnn.cu);
training stays out of scope.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

__all__ = ["Mlp", "IterationWeights", "DssModel", "param_count", "param_arrays",
           "flat_params", "init_model", "save_model", "load_model"]


@dataclass
class Mlp:
    """One-hidden-layer perceptron: relu(x @ w1 + b1) @ w2 + b2 (dss.py:54-61)."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


@dataclass
class IterationWeights:
    phi_out: Mlp  # outgoing-message MLP, input (2d+3)
    phi_in: Mlp   # ingoing-message MLP, input (2d+3)
    psi: Mlp      # latent-update MLP, input (3d+1)
    dec: Mlp      # decoder, input d, output 1


@dataclass
class DssModel:
    k_bar: int
    d: int
    alpha: float
    seed: int
    layers: list

    def n_params(self) -> int:
        return sum(arr.size for arr in param_arrays(self))


def param_count(k_bar: int, d: int) -> int:
    """Closed-form trainable parameter count (dss.py:84-86)."""
    return k_bar * (11 * d * d + 15 * d + 1)


def param_arrays(model: DssModel) -> list:
    """All weight arrays in the canonical (serialization) order (dss.py:93-99)."""
    out = []
    for layer in model.layers:
        for mlp in (layer.phi_out, layer.phi_in, layer.psi, layer.dec):
            out.extend((mlp.w1, mlp.b1, mlp.w2, mlp.b2))
    return out


def flat_params(model: DssModel) -> np.ndarray:
    """Concatenated float64 parameters in canonical order (the C ABI's input)."""
    return np.concatenate([np.ascontiguousarray(a, dtype=np.float64).ravel()
                           for a in param_arrays(model)])


def _xavier_mlp(rng, n_in, n_hidden, n_out) -> Mlp:
    a1 = np.sqrt(6.0 / (n_in + n_hidden))
    w1 = rng.uniform(-a1, a1, (n_in, n_hidden))
    a2 = np.sqrt(6.0 / (n_hidden + n_out))
    w2 = rng.uniform(-a2, a2, (n_hidden, n_out))
    return Mlp(w1, np.zeros(n_hidden), w2, np.zeros(n_out))


def init_model(k_bar: int, d: int, alpha: float = 1e-3, seed: int = 0) -> DssModel:
    """Xavier-uniform weights, zero biases, deterministic per seed (dss.py:110-127)."""
    if k_bar < 1 or d < 1:
        raise ValueError("k_bar and d must be >= 1")
    rng = np.random.default_rng(seed)
    layers = []
    for _ in range(k_bar):
        layers.append(IterationWeights(
            phi_out=_xavier_mlp(rng, 2 * d + 3, d, d),
            phi_in=_xavier_mlp(rng, 2 * d + 3, d, d),
            psi=_xavier_mlp(rng, 3 * d + 1, d, d),
            dec=_xavier_mlp(rng, d, d, 1),
        ))
    model = DssModel(k_bar, d, alpha, seed, layers)
    assert model.n_params() == param_count(k_bar, d)
    return model


def save_model(model: DssModel, path: str) -> None:
    """JSON header line + little-endian float64 blocks (dss.py:530-544)."""
    header = json.dumps({"format": "dss-v1", "k_bar": model.k_bar, "d": model.d,
                         "alpha": model.alpha, "seed": model.seed})
    with open(path, "wb") as fh:
        fh.write(header.encode("ascii") + b"\n")
        for arr in param_arrays(model):
            fh.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def load_model(path: str) -> DssModel:
    """dss-v1 reader with the reference's error messages (dss.py:547-571)."""
    with open(path, "rb") as fh:
        header_line = fh.readline()
        blob = fh.read()
    try:
        header = json.loads(header_line.decode("ascii"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise ValueError(f"malformed model header: {exc}") from exc
    if header.get("format") != "dss-v1":
        raise ValueError(f"unsupported model format {header.get('format')!r}")
    k_bar, d = int(header["k_bar"]), int(header["d"])
    skeleton = init_model(k_bar, d, float(header["alpha"]), seed=int(header["seed"]))
    arrays = param_arrays(skeleton)
    expected = sum(a.size for a in arrays) * 8
    if len(blob) != expected:
        raise ValueError(f"weight block size mismatch: expected {expected} bytes for "
                         f"k_bar={k_bar}, d={d}, got {len(blob)}")
    flat = np.frombuffer(blob, dtype="<f8")
    pos = 0
    for arr in arrays:
        arr[...] = flat[pos: pos + arr.size].reshape(arr.shape)
        pos += arr.size
    return skeleton
