"""Problem containers and result reports: seeded instances and outputs exchanged as files.

Mirrors the reference's instance recipe and container (include/sinktail/problem.hpp:19-99,
src/problem.cpp:8-137) so a problem written by either side loads on the other:

  * ``InstanceSpec`` -- same fields and JSON keys (``L_q, L_k, d, W, T, R, epsilon, schedule, seed,
    dustbin_block, tile_block``; problem.cpp:8-45);
  * ``Support`` -- ``SupportMask::to_json`` / ``from_json`` (src/support.cpp:242-284): kind
    ``banded`` / ``explicit`` / ``augmented``, masks as 0/1 arrays, explicit edge lists;
  * the container file -- magic ``STPC0001``, a little-endian u64 header length, the JSON header
    (``container: "sinktail-problem/1"``, ``spec``, ``support``, ``buffers``: name / rows / cols /
    dtype f64 / offset), then the raw row-major f64 buffers (problem.cpp:47-137).  Buffers other
    than Q, K, V (here the loss cotangent ``G``) are skipped by the reference loader.

Extension (not in the reference): ``save_result`` / ``load_result`` write the outputs of one run in
the same layout (``container: "sinktail-result/1"``, scalars in the header) -- the golden fixtures
under tests/golden/ are pairs of these files.

``run_problem`` runs a container through the device path (one head, B = H = 1).
"""
from __future__ import annotations

import dataclasses
import json
import struct
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

MAGIC = b"STPC0001"


@dataclasses.dataclass
class InstanceSpec:
    """problem.hpp:19-34 (defaults included)."""
    n_rows: int = 64
    n_cols: int = 64
    head_dim: int = 8
    half_band: int = 16
    base_depth: int = 15
    tail_depth: int = 2
    epsilon: float = 1.0
    stages: List[Tuple[float, int]] = dataclasses.field(default_factory=list)  # empty -> single stage
    seed: int = 0
    dustbin_block: int = 0
    tile_block: int = 64

    def to_json(self) -> dict:
        return {"L_q": self.n_rows, "L_k": self.n_cols, "d": self.head_dim, "W": self.half_band,
                "T": self.base_depth, "R": self.tail_depth, "epsilon": self.epsilon,
                "schedule": [[float(e), int(n)] for e, n in self.stages], "seed": self.seed,
                "dustbin_block": self.dustbin_block, "tile_block": self.tile_block}

    @staticmethod
    def from_json(j: dict) -> "InstanceSpec":
        return InstanceSpec(n_rows=int(j["L_q"]), n_cols=int(j["L_k"]), head_dim=int(j["d"]), half_band=int(j["W"]),
                            base_depth=int(j["T"]), tail_depth=int(j["R"]), epsilon=float(j["epsilon"]),
                            stages=[(float(s[0]), int(s[1])) for s in j.get("schedule", [])],
                            seed=int(j["seed"]), dustbin_block=int(j.get("dustbin_block", 0)),
                            tile_block=int(j.get("tile_block", 64)))

    def eps_schedule(self) -> Optional[List[Tuple[float, int]]]:
        return list(self.stages) if self.stages else None

    def final_epsilon(self) -> float:
        return float(self.stages[-1][0]) if self.stages else float(self.epsilon)


@dataclasses.dataclass
class Support:
    """SupportMask as serialised by the reference (src/support.cpp:242-284)."""
    kind: str
    n_rows: int
    n_cols: int
    half_band: int
    row_mask: np.ndarray  # bool [n_rows]
    col_mask: np.ndarray  # bool [n_cols]
    dustbin_block: int = 0
    edges: Optional[np.ndarray] = None  # int64 [E, 2], explicit supports only

    @staticmethod
    def banded(n_rows: int, n_cols: int, half_band: int, row_mask=None, col_mask=None) -> "Support":
        rm = np.ones(n_rows, bool) if row_mask is None else np.asarray(row_mask, bool).copy()
        cm = np.ones(n_cols, bool) if col_mask is None else np.asarray(col_mask, bool).copy()
        if rm.shape != (n_rows,) or cm.shape != (n_cols,):
            raise ValueError("mask sized to the wrong support")
        return Support("banded", n_rows, n_cols, half_band, rm, cm)

    def contains(self, i: int, j: int) -> bool:
        if self.kind == "explicit":
            return bool(np.any((self.edges[:, 0] == i) & (self.edges[:, 1] == j)))
        return bool(abs(i - j) <= self.half_band and self.row_mask[i] and self.col_mask[j])

    def to_json(self) -> dict:
        j = {"kind": self.kind, "L_q": self.n_rows, "L_k": self.n_cols, "W": self.half_band,
             "dustbin_block": self.dustbin_block, "row_mask": [int(b) for b in self.row_mask],
             "col_mask": [int(b) for b in self.col_mask]}
        if self.kind == "explicit":
            j["edges"] = [[int(a), int(b)] for a, b in self.edges]
        return j

    @staticmethod
    def from_json(j: dict) -> "Support":
        kind = j["kind"]
        if kind not in ("banded", "explicit", "augmented"):
            raise ValueError(f"unknown support kind {kind!r}")
        edges = np.asarray(j["edges"], dtype=np.int64).reshape(-1, 2) if kind == "explicit" else None
        return Support(kind, int(j["L_q"]), int(j["L_k"]), int(j.get("W", 0)),
                       np.asarray(j["row_mask"], dtype=np.int64) != 0, np.asarray(j["col_mask"], dtype=np.int64) != 0,
                       int(j.get("dustbin_block", 0)), edges)


@dataclasses.dataclass
class ProblemContainer:
    """problem.hpp:90-96: spec, support and the Q / K / V buffers (f64, row-major); ``extra`` holds
    further named buffers (e.g. the loss cotangent G)."""
    spec: InstanceSpec
    support: Support
    Q: np.ndarray
    K: np.ndarray
    V: np.ndarray
    extra: Dict[str, np.ndarray] = dataclasses.field(default_factory=dict)


def _write(path: str, container: str, header: dict, buffers: Sequence[Tuple[str, np.ndarray]]) -> None:
    payload = bytearray()
    descs = []
    for name, m in buffers:
        m = np.ascontiguousarray(m, dtype="<f8")
        if m.ndim == 1:
            m = m.reshape(1, -1)
        descs.append({"name": name, "rows": int(m.shape[0]), "cols": int(m.shape[1]), "dtype": "f64",
                      "offset": len(payload)})
        payload += m.tobytes()
    h = dict(header)
    h["container"] = container
    h["buffers"] = descs
    text = json.dumps(h, separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<Q", len(text)))
        f.write(text)
        f.write(bytes(payload))


def _read(path: str, container: str) -> Tuple[dict, Dict[str, np.ndarray]]:
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != MAGIC:
        raise ValueError(f"{path} is not a sinktail problem container")
    (hlen,) = struct.unpack("<Q", data[8:16])
    header = json.loads(data[16:16 + hlen].decode())
    if header.get("container") != container:
        raise ValueError(f"{path}: expected a {container} container, found {header.get('container')!r}")
    payload = memoryview(data)[16 + hlen:]
    bufs = {}
    for b in header["buffers"]:
        rows, cols, off = int(b["rows"]), int(b["cols"]), int(b["offset"])
        if b.get("dtype", "f64") != "f64":
            raise ValueError(f"unsupported buffer dtype {b.get('dtype')!r}")
        if off + rows * cols * 8 > len(payload):
            raise ValueError("problem container payload truncated")
        bufs[b["name"]] = np.frombuffer(payload[off: off + rows * cols * 8], dtype="<f8").reshape(rows, cols).copy()
    return header, bufs


def save_problem(path: str, p: ProblemContainer) -> None:
    """problem.cpp:73-103."""
    bufs = [("Q", p.Q), ("K", p.K), ("V", p.V)] + sorted(p.extra.items())
    _write(path, "sinktail-problem/1", {"spec": p.spec.to_json(), "support": p.support.to_json()}, bufs)


def load_problem(path: str) -> ProblemContainer:
    """problem.cpp:105-135."""
    header, bufs = _read(path, "sinktail-problem/1")
    extra = {k: v for k, v in bufs.items() if k not in ("Q", "K", "V")}
    return ProblemContainer(InstanceSpec.from_json(header["spec"]), Support.from_json(header["support"]),
                            bufs["Q"], bufs["K"], bufs["V"], extra)


def save_result(path: str, outputs: Dict[str, np.ndarray], scalars: Dict[str, float], meta: Optional[dict] = None) -> None:
    _write(path, "sinktail-result/1", {"scalars": {k: float(v) for k, v in scalars.items()}, "meta": meta or {}},
           sorted(outputs.items()))


def load_result(path: str) -> Tuple[Dict[str, np.ndarray], Dict[str, float], dict]:
    header, bufs = _read(path, "sinktail-result/1")
    return bufs, {k: float(v) for k, v in header["scalars"].items()}, header.get("meta", {})


def normal_matrix(seed: int, tag: str, rows: int, cols: int, scale: float = 1.0) -> np.ndarray:
    """rng.hpp:46-56 through the library's bit-exact generator (st_normal_fill)."""
    from .configs import normal_fill
    return normal_fill(seed, tag, 0, rows * cols, scale).reshape(rows, cols)


def make_instance(spec: InstanceSpec, row_mask=None, col_mask=None, with_loss: bool = True) -> ProblemContainer:
    """problem.hpp:56-88 for plain banded supports (optionally masked): Q, K, V from tags "Q", "K",
    "V"; with_loss adds the linear loss cotangent G from tag "G", zeroed on inactive rows
    (random_linear_loss, test_util.hpp)."""
    if spec.dustbin_block:
        raise ValueError("the dense augmented dustbin support is not a band; use the spoke dustbin of BandSpec")
    sup = Support.banded(spec.n_rows, spec.n_cols, spec.half_band, row_mask, col_mask)
    p = ProblemContainer(spec, sup, normal_matrix(spec.seed, "Q", spec.n_rows, spec.head_dim),
                         normal_matrix(spec.seed, "K", spec.n_cols, spec.head_dim),
                         normal_matrix(spec.seed, "V", spec.n_cols, spec.head_dim))
    if with_loss:
        G = normal_matrix(spec.seed, "G", spec.n_rows, spec.head_dim)
        G[~active_rows(sup)] = 0.0
        p.extra["G"] = G
    return p


def active_rows(sup: Support) -> np.ndarray:
    """Rows with at least one edge (SupportMask::row_active)."""
    i = np.arange(sup.n_rows)
    lo, hi = np.maximum(0, i - sup.half_band), np.minimum(sup.n_cols - 1, i + sup.half_band)
    cum = np.concatenate([[0], np.cumsum(sup.col_mask)])
    return sup.row_mask & (cum[hi + 1] - cum[lo] > 0)


def band_spec(p: ProblemContainer, dtype: str = "f32"):
    """BandSpec of a container (one head)."""
    from .band import BandSpec
    if p.support.kind != "banded":
        raise ValueError("only banded supports run on the band operator")
    s = p.spec
    return BandSpec(batch=1, heads=1, seq_q=s.n_rows, seq_k=s.n_cols, head_dim=s.head_dim, half_band=s.half_band,
                    base_depth=s.base_depth, tail_depth=s.tail_depth, epsilon=s.final_epsilon(), dtype=dtype,
                    eps_schedule=s.eps_schedule())


def run_problem(p: ProblemContainer, mode: str = "one_reference", device="cuda") -> Dict[str, np.ndarray]:
    """Forward + backward of a container on the device path (f32).  mode: "one_reference",
    "direct_four_plan" or "generic_tail" (any tail depth).  Returns O, dQ, dK, dV, eta_v, d_eps."""
    import torch
    from . import band
    spec = band_spec(p)
    t = lambda x, L: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device).reshape(1, 1, L, -1)
    rm = torch.from_numpy(p.support.row_mask.astype(np.uint8)).to(device).reshape(1, -1)
    cm = torch.from_numpy(p.support.col_mask.astype(np.uint8)).to(device).reshape(1, -1)
    if p.support.row_mask.all() and p.support.col_mask.all():
        rm = cm = None
    run = band.run_surrogate(t(p.Q, spec.seq_q), t(p.K, spec.seq_k), t(p.V, spec.seq_k), spec, rm, cm)
    G = t(p.extra["G"], spec.seq_q)
    cot = band.tail_adjoint(run, G) if mode == "generic_tail" else band.r2_backward(run, G, mode=mode)
    torch.cuda.synchronize()
    mats = {"O": run.output, "dQ": cot.grad_q, "dK": cot.grad_k, "dV": cot.grad_v}
    out = {k: v.cpu().numpy().astype(np.float64).reshape(-1, spec.head_dim) for k, v in mats.items()}
    out["eta_v"] = cot.eta_v.cpu().numpy().astype(np.float64).reshape(-1)
    out["d_eps"] = cot.d_eps.cpu().numpy().astype(np.float64).reshape(-1)
    return out
