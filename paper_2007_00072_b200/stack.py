"""EncoderStack: n post-LN encoder layers (BERT-large: 24) on one GPU, driven through the
layer C ABI -- forward through the stack, backward in reverse, each layer's parameter
gradients ready as soon as its backward is done (the data-parallel all-reduce of layer i
overlaps the backward of layers i-1 .. 0).

Layer i uses dropout subsequences 4*i + site (R5), its own parameters, gradient
buffer and saved activations; the layers share one context and one temporaries buffer.
"""
from __future__ import annotations

from dataclasses import replace

import torch

from .layer import EncoderLayer, LayerCfg
from .ops import Context


class EncoderStack:
    def __init__(self, n_layers: int, dims, dtype: str = "bf16", cfg: LayerCfg | None = None,
                 device=None):
        cfg = cfg or LayerCfg()
        dev = torch.cuda.current_device() if device is None else device
        self.ctx = Context(dev)
        self.layers = []
        scratch = None
        for i in range(n_layers):
            layer = EncoderLayer(dims, dtype, replace(cfg, layer_id=cfg.layer_id + i),
                                 ctx=self.ctx, device=dev, scratch=scratch)
            scratch = layer.scratch
            self.layers.append(layer)
        first = self.layers[0]
        shape = (dims.B, dims.J, first.I)
        # activations between layers (the input of layer i is kept for its backward)
        self.acts = [torch.empty(shape, dtype=first.tdt, device=first.device)
                     for _ in range(n_layers + 1)]
        self.grads_io = [torch.empty(shape, dtype=first.tdt, device=first.device)
                         for _ in range(2)]

    def set_params(self, params_per_layer):
        for layer, prm in zip(self.layers, params_per_layer):
            layer.set_params(prm)

    def forward(self, X: torch.Tensor, mask_bias=None) -> torch.Tensor:
        self.acts[0].copy_(X)
        for i, layer in enumerate(self.layers):
            layer.forward(self.acts[i], mask_bias, self.acts[i + 1])
        return self.acts[-1]

    def backward(self, dY: torch.Tensor, on_layer_done=None) -> torch.Tensor:
        """on_layer_done(i, layer): called after layer i's backward is enqueued (its gradient
        buffer is then final on the stream), e.g. to start its all-reduce."""
        g = dY
        for i in reversed(range(len(self.layers))):
            out = self.grads_io[i % 2]
            self.layers[i].backward(self.acts[i], g, out)
            if on_layer_done is not None:
                on_layer_done(i, self.layers[i])
            g = out
        return g

    def init_optimizer(self):
        """AdamW state (fp32 master parameters, moments) for every layer."""
        for layer in self.layers:
            layer.init_optimizer()

    def optimizer_step(self, lr=1e-4, betas=(0.9, 0.999), eps=1e-6, weight_decay=0.01,
                       stream=None):
        """enc_adamw_step for every layer (one launch each)."""
        for layer in self.layers:
            layer.optimizer_step(lr, betas, eps, weight_decay, stream=stream)

    def train_step(self, X, dY, lr=1e-4, reduce=None, mask_bias=None):
        """One training step: forward, backward, AdamW.  reduce(layer), if given, is called
        once a layer's gradients are final (e.g. the data-parallel all-reduce); work handles it
        returns (async collectives) are waited on before the parameters are updated."""
        self.forward(X, mask_bias)
        works = []

        def done(i, layer):
            w = reduce(layer)
            if w is not None:   # asynchronous collectives: waited on before the update
                works.extend(w if isinstance(w, (list, tuple)) else [w])
        self.backward(dY, on_layer_done=None if reduce is None else done)
        for w in works:
            w.wait()
        self.optimizer_step(lr)

    def step_host(self, X_host, dY_host, Y_host, dX_host, mask_bias=None, stream=None):
        """One training step from host memory: H2D X and dY (pinned host tensors), forward
        and backward through every layer, D2H the output Y and the input gradient dX."""
        s = stream or torch.cuda.current_stream(self.layers[0].device)
        with torch.cuda.stream(s):
            self.acts[0].copy_(X_host, non_blocking=True)
            dY = self.grads_io[len(self.layers) % 2]   # layer n-1 writes the other one
            dY.copy_(dY_host, non_blocking=True)
            for i, layer in enumerate(self.layers):
                layer.forward(self.acts[i], mask_bias, self.acts[i + 1], stream=s)
            Y_host.copy_(self.acts[-1], non_blocking=True)
            g = dY
            for i in reversed(range(len(self.layers))):
                out = self.grads_io[i % 2]
                self.layers[i].backward(self.acts[i], g, out, stream=s)
                g = out
            dX_host.copy_(g, non_blocking=True)
