"""Weight declaration, seeded initialisation and the EGN1 container.

The weight names, shapes (out, in), declaration order and the
SeedSequence-per-array U(+-1/sqrt(fan_in)) initialisation are the drop-in
contract of egn/params.py:30-108; the EGN1 binary layout (magic, nine u32
header words, raw little-endian f64 blobs) is egn/params.py:1-6,120-162.
Host-side numpy (fp64) is the canonical parameter store, exactly as in the
reference; the model copies it to fp32 device buffers.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .config import DIMENET, GEMNET, ModelConfig

MAX_Z = 118
MAGIC = b"EGN1"
_CODE = {DIMENET: 0, GEMNET: 1}
_VARIANT = {v: k for k, v in _CODE.items()}


@dataclass(frozen=True)
class ParamSpec:
    name: str
    shape: tuple[int, ...]
    fan_in: int


def _block_specs(c: ModelConfig, b: int) -> list[ParamSpec]:
    p = f"block{b}."
    kl = c.k_rbf * c.l_sbf
    out = [
        ParamSpec(p + "tu.down", (c.d_t, c.d_e), c.d_e),
        ParamSpec(p + "tu.rbf_gate", (c.d_t, c.k_rbf), c.k_rbf),
        ParamSpec(p + "tu.sbf_gate", (c.d_t, kl), kl),
    ]
    if c.variant == GEMNET:
        out += [
            ParamSpec(p + "tu.bilinear_a", (c.d_bil, c.d_t), c.d_t),
            ParamSpec(p + "tu.bilinear_b", (c.d_bil, c.d_t), c.d_t),
            ParamSpec(p + "tu.bilinear_proj", (c.d_t, c.d_bil), c.d_bil),
        ]
    out.append(ParamSpec(p + "tu.up", (c.d_e, c.d_t), c.d_t))
    for stage, d_out, d_in in (("eu", c.d_e, 2 * c.d_e), ("nu", c.d_v, c.d_e)):
        d_hidden = d_out
        out += [
            ParamSpec(f"{p}{stage}.w1", (d_hidden, d_in), d_in),
            ParamSpec(f"{p}{stage}.b1", (d_hidden,), d_in),
            ParamSpec(f"{p}{stage}.w2", (d_out, d_hidden), d_hidden),
            ParamSpec(f"{p}{stage}.b2", (d_out,), d_hidden),
        ]
    if c.variant == GEMNET:
        d_in = c.d_e + c.d_v
        out += [
            ParamSpec(p + "eu2.w1", (c.d_e, d_in), d_in),
            ParamSpec(p + "eu2.b1", (c.d_e,), d_in),
            ParamSpec(p + "eu2.w2", (c.d_e, c.d_e), c.d_e),
            ParamSpec(p + "eu2.b2", (c.d_e,), c.d_e),
            ParamSpec(p + "sym.w", (c.d_e, c.d_e), c.d_e),
        ]
    out += [
        ParamSpec(p + "gu.w1", (c.d_u, c.d_v), c.d_v),
        ParamSpec(p + "gu.b1", (c.d_u,), c.d_v),
        ParamSpec(p + "gu.w2", (c.d_u, c.d_u), c.d_u),
        ParamSpec(p + "gu.b2", (c.d_u,), c.d_u),
    ]
    return out


def param_specs(config: ModelConfig) -> list[ParamSpec]:
    """All weights in declaration (= serialisation) order."""
    c = config
    specs = [
        ParamSpec("atom_embedding", (MAX_Z, c.d_v), 1),
        ParamSpec("edge_init.w", (c.d_e, c.k_rbf), c.k_rbf),
        ParamSpec("edge_init.b", (c.d_e,), c.k_rbf),
    ]
    for b in range(c.blocks):
        specs += _block_specs(c, b)
    specs += [ParamSpec("energy_head.w", (1, c.d_u), c.d_u), ParamSpec("energy_head.b", (1,), c.d_u)]
    if c.variant == GEMNET:
        specs.append(ParamSpec("force_head.w", (1, c.d_e), c.d_e))
    return specs


@dataclass(frozen=True)
class ModelParams:
    config: ModelConfig
    arrays: dict  # name -> float64 ndarray, declaration order

    def num_params(self) -> int:
        return sum(a.size for a in self.arrays.values())

    def validate(self) -> None:
        specs = param_specs(self.config)
        if [s.name for s in specs] != list(self.arrays):
            raise ValueError("parameter names do not match the declared layout")
        for s in specs:
            a = self.arrays[s.name]
            if a.shape != s.shape or a.dtype != np.float64:
                raise ValueError(f"{s.name}: expected float64 {s.shape}, got {a.dtype} {a.shape}")

    def map_arrays(self, fn) -> dict:
        return {k: fn(v) for k, v in self.arrays.items()}


def init_params(config: ModelConfig) -> ModelParams:
    specs = param_specs(config)
    streams = np.random.SeedSequence(config.seed).spawn(len(specs))
    arrays = {}
    for spec, seq in zip(specs, streams):
        bound = 1.0 / np.sqrt(spec.fan_in)
        arrays[spec.name] = np.random.default_rng(seq).uniform(-bound, bound, size=spec.shape)
    return ModelParams(config, arrays)


def zero_params(config: ModelConfig) -> ModelParams:
    return ModelParams(config, {s.name: np.zeros(s.shape) for s in param_specs(config)})


def save_params(params: ModelParams, path) -> None:
    c = params.config
    params.validate()
    head = struct.pack("<9I", c.blocks, c.d_u, c.d_v, c.d_e, c.d_t, c.d_bil, c.k_rbf, c.l_sbf,
                       _CODE[c.variant])
    with open(path, "wb") as fh:
        fh.write(MAGIC + head)
        for a in params.arrays.values():
            fh.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def load_params(path, cutoff: float = 1.5, seed: int = 0, workers: int = 1) -> ModelParams:
    blob = open(path, "rb").read()
    if blob[:4] != MAGIC:
        raise ValueError(f"bad magic bytes {blob[:4]!r}")
    h = struct.unpack("<9I", blob[4:40])
    if h[8] not in _VARIANT:
        raise ValueError(f"unknown variant code {h[8]}")
    config = ModelConfig(variant=_VARIANT[h[8]], blocks=h[0], d_u=h[1], d_v=h[2], d_e=h[3],
                         d_t=h[4], d_bil=h[5], k_rbf=h[6], l_sbf=h[7], cutoff=cutoff, seed=seed,
                         workers=workers)
    arrays, off = {}, 40
    for s in param_specs(config):
        end = off + 8 * int(np.prod(s.shape, dtype=np.int64))
        if end > len(blob):
            raise ValueError("container truncated")
        arrays[s.name] = np.frombuffer(blob[off:end], dtype="<f8").reshape(s.shape).astype(np.float64)
        off = end
    if off != len(blob):
        raise ValueError("container has trailing bytes")
    return ModelParams(config, arrays)
