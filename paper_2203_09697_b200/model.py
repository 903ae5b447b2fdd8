"""nn.Module face of the model: ``EGNModel(config).forward(batch) -> (energy, forces)``.

Parameters are registered under the reference's weight names
(egn/params.py:30-70, e.g. ``block0.tu.down``), so ``state_dict()`` keys
equal ``param_specs`` names; they are views into one flat fp32 device
buffer.  The forward/backward run the native engine (engine.py) behind the custom op
``torch.ops.egn.energy_forces`` (torch_ops.py) and its registered autograd formula, so
the model is visible to the dispatcher, FakeTensor tracing and torch.compile.
"""

from __future__ import annotations

import torch

from .config import GEMNET, ModelConfig
from .engine import DeviceWeights, Engine
from .graph import BatchGraph, build_batch
from .params import ModelParams, init_params


class EGNModel(torch.nn.Module):
    def __init__(self, config: ModelConfig, params: ModelParams | None = None, device="cuda"):
        super().__init__()
        self.config = config
        params = params if params is not None else init_params(config)
        self.weights = DeviceWeights.from_params(params, device)
        self.engine = Engine(self.weights)
        self._names = []
        for spec in self.weights.specs:
            *path, leaf = spec.name.split(".")
            mod = self
            for part in path:
                if not hasattr(mod, part):
                    mod.add_module(part, torch.nn.Module())
                mod = getattr(mod, part)
            mod.register_parameter(leaf, torch.nn.Parameter(self.weights.w[spec.name], requires_grad=True))
            self._names.append(spec.name)

    def parameters_in_order(self):
        params = dict(self.named_parameters())
        return [params[n] for n in self._names]

    def batch(self, systems) -> BatchGraph:
        return build_batch(systems, self.config.cutoff, device=self.weights.flat.device)

    def _key(self, bg: BatchGraph) -> int:
        """Registry key of (engine, batch) for egn::energy_forces; the last few batches stay
        registered (the graph topology is built outside the traced region)."""
        from .torch_ops import register_model, release_model

        keys = self.__dict__.setdefault("_op_keys", {})
        ent = keys.get(id(bg))
        if ent is None or ent[1] is not bg:
            while len(keys) >= 4:
                old = next(iter(keys))
                release_model(keys.pop(old)[0])
            ent = (register_model(self.engine, bg), bg)
            keys[id(bg)] = ent
        return ent[0]

    def forward(self, batch):
        """batch: BatchGraph, AtomicSystem or list of systems -> (energy [G], forces [V, 3])."""
        from . import torch_ops  # noqa: F401  (registers torch.ops.egn.*)

        bg = batch if isinstance(batch, BatchGraph) else self.batch(batch)
        return torch.ops.egn.energy_forces(self.parameters_in_order(), bg.pos, bg.graph_ptr, self._key(bg))

    def to_params(self) -> ModelParams:
        return ModelParams(self.config, self.weights.to_numpy())
