"""CUDA-graph captured steps for steady-state serving.

A background model is rebuilt and frames are classified batch after batch
with fixed shapes, so the whole device work of a step -- build (K1 build,
K2 pyramid, K3 merge) and classify (K4) -- is captured once into CUDA graphs
and replayed: no per-launch host work, no launch gaps.  Inputs live in static
device buffers (copy new frames into ``train`` / ``test`` before a replay);
outputs are the static ``model`` / ``masks``.
"""

from __future__ import annotations

from . import _device
from .detect import classify
from .model import BackgroundModel, ModelConfig, build_background_model_device


class CapturedStep:
    """Build-from-``train`` + classify-``test`` as two replayable CUDA graphs."""

    def __init__(self, train, test, config: ModelConfig, packed: bool = False, warmup: int = 2):
        t = _device.torch()
        self.train, self.test, self.config = train, test, config
        n, h, w = int(test.shape[0]), int(test.shape[1]), int(test.shape[2])
        shape = (n, (h * w + 7) // 8) if packed else (n, h, w)
        self.masks = t.empty(shape, dtype=t.uint8, device=test.device)
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(side):          # warm-up: one-time attribute / occupancy setup
            for _ in range(warmup):
                m = build_background_model_device(train, config)
                classify(m, test, out=self.masks, packed=packed)
        t.cuda.current_stream().wait_stream(side)
        t.cuda.synchronize()
        self.build_graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.build_graph):
            self.model: BackgroundModel = build_background_model_device(train, config)
        self.classify_graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.classify_graph):
            classify(self.model, test, out=self.masks, packed=packed)
        t.cuda.synchronize()

    def build(self) -> BackgroundModel:
        self.build_graph.replay()
        return self.model

    def classify(self):
        self.classify_graph.replay()
        return self.masks

    def step(self):
        self.build_graph.replay()
        self.classify_graph.replay()
        return self.masks
