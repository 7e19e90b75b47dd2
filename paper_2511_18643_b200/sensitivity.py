"""Per-channel quantization sensitivity and boost-rate sweeps on the device.

The reference's desk-scale experiments (analysis.py:47-236) that justify the
Dynamic Channel-wise Precision Boost: how much the attention probabilities
move when one key channel is quantized to 2 bits (``channel_sensitivity``),
and how much boosting a selection of channels to 4 bits recovers
(``attention_mse``, ``boost_sweep``, ``boost_sweep_experiment``).  Same names,
arguments, return types and errors as ``kittykv.analysis``; the fp64 numerics
run in libkitty_b200.so (csrc/kitty_analysis.cu: kitty_channel_sensitivity,
kitty_attention_mse); channel scores and the magnitude selection use the
device codec (kitty_channel_scores / kitty_select_boost).  The host only
draws the ``random`` baseline's selections and the synthetic data from
numpy's PCG64, exactly as the reference does (quant.py:95-97,
tensor_io.py:119-124), so both heuristics see identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import PASSTHROUGH_BITS
from .errors import KittyError, TensorIOError
from .pages import _device, _stream, channel_scores, select_boost


def _stack_heads(x, what: str) -> np.ndarray:
    """analysis.py:38-44."""
    x = np.asarray(x, dtype=np.float32)
    if x.ndim == 2:
        x = x[None]
    if x.ndim != 3:
        raise KittyError(f"{what} must be (heads, tokens, channels) or 2-D")
    return x


def _ws(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=_device())


@dataclass(frozen=True)
class SensitivityReport:
    """Attention-probability MSE of quantizing each key channel alone (analysis.py:50-60)."""

    mse: np.ndarray  # (h_q, D) float64
    ranking: np.ndarray  # (h_q, D) channels by descending MSE per head
    mean_mse: np.ndarray  # (D,) mean across query heads

    def top_channels(self, k: int) -> np.ndarray:
        """The k channels with the largest head-averaged MSE."""
        return np.argsort(-self.mean_mse, kind="stable")[:k]


def channel_sensitivity(queries, keys, bits: int = 2) -> SensitivityReport:
    """analysis.py:63-104 on the device: for every query head and key channel,
    the MSE between the baseline and the perturbed (lq x L) probability
    matrices when that channel alone is fake-quantized per channel at ``bits``
    (a rank-1 logit update), in fp64.  ``bits=16`` is the identity (zeros)."""
    queries = _stack_heads(queries, "queries")
    keys = _stack_heads(keys, "keys")
    h_q, lq, d = queries.shape
    h_kv, length, dk = keys.shape
    if d != dk:
        raise KittyError("queries and keys disagree on the channel count")
    if h_q % h_kv != 0:
        raise KittyError("query head count must be a multiple of KV head count")
    if bits == PASSTHROUGH_BITS or lq == 0 or length == 0:
        mse = np.zeros((h_q, d), dtype=np.float64)
        ranking = np.tile(np.arange(d), (h_q, 1)) if bits == PASSTHROUGH_BITS else np.argsort(-mse, axis=1, kind="stable")
        return SensitivityReport(mse=mse, ranking=ranking, mean_mse=mse.mean(axis=0))
    lib = _lib.load_library()
    dev = _device()
    qt = torch.from_numpy(np.ascontiguousarray(queries)).to(dev)
    kt = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    out = torch.empty((h_q, d), dtype=torch.float64, device=dev)
    ws = _ws(lib.kitty_sensitivity_workspace_bytes(h_q, lq, h_kv, length, d))
    _lib.check(lib.kitty_channel_sensitivity(qt.data_ptr(), h_q, lq, kt.data_ptr(), h_kv, length, d, int(bits),
                                             out.data_ptr(), ws.data_ptr(), ws.numel(), _stream()),
               "channel_sensitivity")
    mse = out.cpu().numpy()
    ranking = np.argsort(-mse, axis=1, kind="stable")
    return SensitivityReport(mse=mse, ranking=ranking, mean_mse=mse.mean(axis=0))


@dataclass(frozen=True)
class SweepRow:
    """analysis.py:110-116."""

    fraction: float
    heuristic: str
    mean_mse: float
    max_deviation: float
    runs: int


def attention_mse(keys, queries, selection) -> float:
    """analysis.py:119-142 on the device: selected key channels fake-quantized
    at 4 bits, the rest at 2, attention-probability MSE against full
    precision, averaged over query heads."""
    keys = np.asarray(keys, dtype=np.float32)
    queries = _stack_heads(queries, "queries")
    if keys.ndim != 2:
        raise KittyError("keys must be (tokens, channels)")
    length, d = keys.shape
    heads, lq, dq = queries.shape
    if dq != d:
        raise KittyError("queries and keys disagree on the channel count")
    widths = np.full(d, 2, dtype=np.int32)
    widths[np.asarray(selection, dtype=np.int64)] = 4
    lib = _lib.load_library()
    dev = _device()
    kt = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    qt = torch.from_numpy(np.ascontiguousarray(queries)).to(dev)
    bt = torch.from_numpy(widths).to(dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    ws = _ws(lib.kitty_attention_mse_workspace_bytes(heads, lq, length, d))
    _lib.check(lib.kitty_attention_mse(kt.data_ptr(), length, d, qt.data_ptr(), heads, lq, bt.data_ptr(),
                                       out.data_ptr(), ws.data_ptr(), ws.numel(), _stream()), "attention_mse")
    return float(out.item())


def boost_sweep(keys, queries, fractions, heuristics=("magnitude", "random"), random_draws: int = 5,
                seed: int = 0) -> list[SweepRow]:
    """analysis.py:145-186: attention MSE per (boost fraction, heuristic).
    Magnitude selection on the device; the random baseline's draws come from
    the seeded PCG64 generator in the reference's order."""
    keys = np.asarray(keys, dtype=np.float32)
    scores = channel_scores(keys)
    rng = np.random.default_rng(seed)
    rows = []
    for fraction in fractions:
        for heuristic in heuristics:
            if heuristic == "magnitude":
                sel = select_boost(scores, fraction, "magnitude")
                runs = [attention_mse(keys, queries, sel.boosted)]
            elif heuristic == "random":
                runs = []
                for _ in range(random_draws):
                    sel = select_boost(scores, fraction, "random", rng)
                    runs.append(attention_mse(keys, queries, sel.boosted))
            else:
                raise KittyError(f"unknown heuristic {heuristic!r}")
            mean = float(np.mean(runs))
            rows.append(SweepRow(fraction=float(fraction), heuristic=heuristic, mean_mse=mean,
                                 max_deviation=float(np.max(np.abs(np.asarray(runs) - mean))), runs=len(runs)))
    return rows


@dataclass(frozen=True)
class SyntheticSpec:
    """tensor_io.py:89-117: a (tokens, channels) Gaussian matrix with a few
    high-magnitude channels."""

    tokens: int
    channels: int
    outlier_channels: tuple = field(default_factory=tuple)
    outlier_gain: float = 1.0
    base_std: float = 1.0
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "outlier_channels", tuple(self.outlier_channels))
        if self.tokens < 0 or self.channels < 0:
            raise TensorIOError("tokens and channels must be non-negative")
        if len(set(self.outlier_channels)) != len(self.outlier_channels):
            raise TensorIOError("outlier channel indices must be unique")
        if any(not 0 <= c < self.channels for c in self.outlier_channels):
            raise TensorIOError("outlier channel index out of range")
        if self.outlier_gain < 1.0:
            raise TensorIOError("outlier_gain must be >= 1.0")
        if not self.base_std > 0:
            raise TensorIOError("base_std must be positive")


def generate_synthetic(spec: SyntheticSpec) -> np.ndarray:
    """tensor_io.py:119-124 (host numpy PCG64: the experiment's input data)."""
    rng = np.random.default_rng(spec.seed)
    m = rng.normal(0.0, spec.base_std, size=(spec.tokens, spec.channels))
    if spec.outlier_channels:
        m[:, list(spec.outlier_channels)] *= spec.outlier_gain
    return m.astype(np.float32)


def boost_sweep_experiment(fractions, n_seeds: int = 20, tokens: int = 1024, channels: int = 128,
                           outlier_channels=(3, 17), outlier_gain: float = 8.0, base_std: float = 1.0,
                           query_tokens: int = 64, heuristics=("magnitude", "random"), seed: int = 0) -> list[SweepRow]:
    """analysis.py:189-236: the sweep over freshly generated synthetic datasets,
    per-seed MSEs averaged with the maximum observed deviation."""
    per_cell = {(float(f), h): [] for f in fractions for h in heuristics}
    for s in range(n_seeds):
        spec = SyntheticSpec(tokens=tokens, channels=channels, outlier_channels=tuple(outlier_channels),
                             outlier_gain=outlier_gain, base_std=base_std, seed=seed + s)
        keys = generate_synthetic(spec)
        q_rng = np.random.default_rng((seed + s, 113))
        queries = q_rng.normal(0.0, 1.0, size=(query_tokens, channels)).astype(np.float32)
        for row in boost_sweep(keys, queries, fractions, heuristics, random_draws=1, seed=seed + s):
            per_cell[(row.fraction, row.heuristic)].append(row.mean_mse)
    rows = []
    for (fraction, heuristic), runs in per_cell.items():
        mean = float(np.mean(runs))
        rows.append(SweepRow(fraction=fraction, heuristic=heuristic, mean_mse=mean,
                             max_deviation=float(np.max(np.abs(np.asarray(runs) - mean))), runs=len(runs)))
    return rows
