"""nn.Module face of the model: ``EGNModel(config).forward(batch) -> (energy, forces)``.

Parameters are registered under the reference's weight names
(egn/params.py:30-70, e.g. ``block0.tu.down``), so ``state_dict()`` keys
equal ``param_specs`` names; they are views into one flat fp32 device
buffer.  The forward/backward run the native engine (engine.py); the
autograd Function only routes gradients, it never records torch ops.
"""

from __future__ import annotations

import torch

from .config import GEMNET, ModelConfig
from .engine import DeviceWeights, Engine
from .graph import BatchGraph, build_batch
from .params import ModelParams, init_params


class _EGNFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, engine: Engine, bg: BatchGraph, *params):
        fw = engine.forward(bg)
        if engine.config.variant == GEMNET:
            forces = fw.forces
        else:
            # energy-centric forces F = -dE/dx at fixed topology (tasks.py:57-59)
            ones = torch.ones(bg.num_graphs, device=bg.device)
            forces = (-engine.backward(bg, fw, ones)).to(torch.float32)
        ctx.engine, ctx.bg, ctx.fw = engine, bg, fw
        ctx.mark_non_differentiable(forces) if engine.config.variant != GEMNET else None
        return fw.energy.clone(), forces

    @staticmethod
    def backward(ctx, g_energy, g_forces):
        engine, bg, fw = ctx.engine, ctx.bg, ctx.fw
        gem = engine.config.variant == GEMNET
        if g_energy is None:
            g_energy = torch.zeros(bg.num_graphs, device=bg.device)
        if not gem:
            g_forces = None  # non-differentiable output (tasks.py:147-151)
        engine.backward(bg, fw, g_energy, g_forces)
        w = engine.weights
        grads = tuple(w.g[s.name].clone() for s in w.specs)
        return (None, None) + grads


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

    def forward(self, batch):
        """batch: BatchGraph, AtomicSystem or list of systems -> (energy [G], forces [V, 3])."""
        bg = batch if isinstance(batch, BatchGraph) else self.batch(batch)
        return _EGNFunction.apply(self.engine, bg, *self.parameters_in_order())

    def to_params(self) -> ModelParams:
        return ModelParams(self.config, self.weights.to_numpy())
