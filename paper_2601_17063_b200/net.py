"""EvictionNet parameters and the .evnet checkpoint container.

Mirrors pkg/src/moecache/net.py:18-105, 282-332: the same parameter names and
shapes (w1[H][2E] b1[H] w2[H][H] b2[H] w3[E][H] b3[E], float64), the same
seeded uniform(+-1/sqrt(fan_in)) initialisation so ``EvictionNet(E, seed=s)``
is bit-identical to the reference's, and the same checkpoint bytes.  The B200
engine consumes the parameters (converted once per call to the transposed
device layout of K3); it never calls ``forward`` -- that host helper exists
only for API compatibility.  Training (net.py:107-279) is train.py's GPU
implementation (K10).
"""
from __future__ import annotations

import json
from typing import Optional

import numpy as np

HIDDEN_SIZE = 128
NUM_LINEAR_LAYERS = 3
ACTIVATION = "silu"
CHECKPOINT_FORMAT_VERSION = 1
PARAM_NAMES = ("w1", "b1", "w2", "b2", "w3", "b3")
_MAGIC = b"EVNET\n"


class NetError(Exception):
    pass


class ShapeMismatchError(NetError):
    pass


class EvictionNet:
    """Per-layer scorer: input 2E features, output E scores."""

    def __init__(self, num_experts: int, hidden: int = HIDDEN_SIZE, seed: int = 0, zero_init: bool = False):
        self.num_experts = int(num_experts)
        self.hidden = int(hidden)
        E, H = self.num_experts, self.hidden
        shapes = (("w1", (H, 2 * E)), ("b1", (H,)), ("w2", (H, H)), ("b2", (H,)), ("w3", (E, H)), ("b3", (E,)))
        self.params: dict[str, np.ndarray] = {}
        rng = None if zero_init else np.random.default_rng(seed)
        fan_in = {"w1": 2 * E, "b1": 2 * E, "w2": H, "b2": H, "w3": H, "b3": H}
        for name, shape in shapes:
            if rng is None:
                self.params[name] = np.zeros(shape)
            else:
                bound = 1.0 / np.sqrt(fan_in[name])
                self.params[name] = rng.uniform(-bound, bound, size=shape)

    def flat_params(self) -> np.ndarray:
        """float64 params in .evnet order (the layout mcb_nets expects)."""
        return np.concatenate([np.ascontiguousarray(self.params[n], dtype=np.float64).ravel()
                               for n in PARAM_NAMES])

    def parameter_count(self) -> int:
        return sum(v.size for v in self.params.values())

    def clone(self) -> "EvictionNet":
        other = EvictionNet(self.num_experts, self.hidden, zero_init=True)
        other.params = {k: v.copy() for k, v in self.params.items()}
        return other

    def forward(self, x: np.ndarray) -> np.ndarray:
        """Host forward for API compatibility (not used by the engine)."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape[-1] != 2 * self.num_experts:
            raise ShapeMismatchError(f"feature length {x.shape[-1]} != 2*num_experts ({2 * self.num_experts})")
        p = self.params

        def silu(z):
            out = np.empty_like(z)
            pos = z >= 0
            out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
            ez = np.exp(z[~pos])
            out[~pos] = ez / (1.0 + ez)
            return z * out

        h = silu(np.atleast_2d(x) @ p["w1"].T + p["b1"])
        h = silu(h @ p["w2"].T + p["b2"])
        out = h @ p["w3"].T + p["b3"]
        return out[0] if x.ndim == 1 else out


def save_net(net: EvictionNet, path) -> int:
    header = {
        "format_version": CHECKPOINT_FORMAT_VERSION,
        "num_experts": net.num_experts,
        "hidden_size": net.hidden,
        "num_linear_layers": NUM_LINEAR_LAYERS,
        "activation": ACTIVATION,
        "dtype": "<f8",
        "params": [[name, list(net.params[name].shape)] for name in PARAM_NAMES],
    }
    blob = _MAGIC + (json.dumps(header, separators=(",", ":")) + "\n").encode("utf-8")
    blob += b"".join(np.ascontiguousarray(net.params[n], dtype="<f8").tobytes() for n in PARAM_NAMES)
    with open(path, "wb") as fh:
        fh.write(blob)
    return len(blob)


def load_net(path, num_experts: Optional[int] = None) -> EvictionNet:
    with open(path, "rb") as fh:
        blob = fh.read()
    if not blob.startswith(_MAGIC):
        raise NetError(f"{path}: not an eviction-net checkpoint")
    end = blob.index(b"\n", len(_MAGIC))
    header = json.loads(blob[len(_MAGIC):end].decode("utf-8"))
    if header.get("format_version") != CHECKPOINT_FORMAT_VERSION:
        raise NetError(f"unsupported checkpoint format version {header.get('format_version')}")
    if num_experts is not None and header["num_experts"] != num_experts:
        raise ShapeMismatchError(f"checkpoint was trained for num_experts={header['num_experts']}, "
                                 f"expected {num_experts}")
    net = EvictionNet(header["num_experts"], header["hidden_size"], zero_init=True)
    off = end + 1
    for name, shape in header["params"]:
        size = int(np.prod(shape)) * 8
        net.params[name] = np.frombuffer(blob[off:off + size], dtype="<f8").astype(np.float64).reshape(shape)
        off += size
    if off != len(blob):
        raise NetError(f"{path}: trailing bytes after parameter arrays")
    return net
