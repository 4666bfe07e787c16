"""CUDA-graph captured steps for steady-state serving.

A background model is rebuilt and frames are classified batch after batch
with fixed shapes, so the whole device work of a step -- build (K1 build,
K2 pyramid, K3 merge) and classify (K4) -- is captured once into CUDA graphs
and replayed: no per-launch host work, no launch gaps.  Inputs live in static
device buffers (copy new frames into ``train`` / ``test`` before a replay);
outputs are the static ``model`` / ``masks``.
"""

from __future__ import annotations

from . import _device, _lib
from .detect import classify
from .model import BackgroundModel, ModelConfig, build_background_model_device, new_workspace


class CapturedStep:
    """Build-from-``train`` + classify-``test`` as replayable CUDA graphs: the
    two halves separately (build / classify, for per-phase timing) and the
    whole step as one graph (step).

    Each graph owns its build workspace (allocated here, referenced for the
    life of the graph), so a replay never shares scratch with an eager build
    or with the other graph.  ``build()`` / ``step()`` return a NEW
    :class:`BackgroundModel` view of the graph's static device buffers, so
    host views (``trees``, ``to_bytes``, ``write_model``) always read the
    replay just done; a returned model is valid until its graph replays again.
    """

    def __init__(self, train, test, config: ModelConfig, packed: bool = False, warmup: int = 2):
        t = _device.torch()
        self.train, self.test, self.config = train, test, config
        n, h, w = int(test.shape[0]), int(test.shape[1]), int(test.shape[2])
        shape = (n, (h * w + 7) // 8) if packed else (n, h, w)
        self.masks = t.empty(shape, dtype=t.uint8, device=test.device)
        n_groups = min(int(train.shape[0]), config.training_frames) // config.group_size
        ws_bytes = _lib.load().obg_build_workspace_bytes(n_groups, config.grid_rows * config.grid_cols,
                                                          config.levels)
        self._ws_build, self._ws_step = new_workspace(ws_bytes), new_workspace(ws_bytes)
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(side):          # warm-up: one-time attribute / occupancy setup
            for _ in range(warmup):
                m = build_background_model_device(train, config, workspace=self._ws_build)
                classify(m, test, out=self.masks, packed=packed)
        t.cuda.current_stream().wait_stream(side)
        t.cuda.synchronize()
        self.build_graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.build_graph):
            self._build_bufs = build_background_model_device(train, config, workspace=self._ws_build)
        self.classify_graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.classify_graph):
            classify(self._build_bufs, test, out=self.masks, packed=packed)
        # the whole step as ONE graph (no launch gap between build and
        # classify); it owns its own model buffers and workspace
        self.step_graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.step_graph):
            self._step_bufs = build_background_model_device(train, config, workspace=self._ws_step)
            classify(self._step_bufs, test, out=self.masks, packed=packed, after_build=True)
        t.cuda.synchronize()
        self._last = self._view(self._build_bufs)

    @staticmethod
    def _view(bufs: BackgroundModel) -> BackgroundModel:
        return BackgroundModel(bufs.config, frame_width=bufs.frame_width, frame_height=bufs.frame_height,
                               _device_pyramids=bufs._dev_pyr, _device_cube=bufs._dev_cube)

    @property
    def model(self) -> BackgroundModel:
        """The model of the most recent replay (build() or step())."""
        return self._last

    def build(self) -> BackgroundModel:
        self.build_graph.replay()
        self._last = self._view(self._build_bufs)
        return self._last

    def classify(self):
        """Classify with the model of the last build()."""
        self.classify_graph.replay()
        return self.masks

    def step(self):
        """Build + classify as one graph replay (model: ``self.model``)."""
        self.step_graph.replay()
        self._last = self._view(self._step_bufs)
        return self.masks


def process_batches(train_host, test_host, config: ModelConfig, out_host=None, chunk: int = 32,
                    packed: bool = False):
    """Host frames in, host masks out, with copies overlapped with the kernels.

    ``train_host`` / ``test_host`` are (n, h, w, 3) uint8 CPU tensors (pinned
    memory gives asynchronous copies).  The training frames go up first and
    the model is built; meanwhile the test frames stream up chunk by chunk on
    a copy stream, each chunk is classified as soon as it lands and its masks
    stream back on a third stream -- H2D, compute and D2H overlap, so the
    batch costs about max(H2D, D2H) over PCIe instead of their sum.
    Returns (model, masks) with masks in ``out_host`` (allocated pinned if
    None): (n, h, w) uint8 0/1, or bit-packed with ``packed``.
    """
    t = _device.torch()
    dev = t.device("cuda", t.cuda.current_device())
    main = t.cuda.current_stream()
    up = t.cuda.Stream()
    with t.cuda.stream(up):
        train = train_host.to(dev, non_blocking=True)
    main.wait_stream(up)
    train.record_stream(main)
    model = build_background_model_device(train, config)
    return model, classify_host(model, test_host, out_host=out_host, chunk=chunk, packed=packed, up=up)


def classify_host(model: BackgroundModel, test_host, out_host=None, chunk: int = 32, packed: bool = False, up=None):
    """Masks of host frames with H2D / classify / D2H overlapped chunk by chunk
    (see ``process_batches``).  Returns ``out_host`` (pinned if allocated here);
    the copies are complete when the current stream is."""
    t = _device.torch()
    dev = t.device("cuda", t.cuda.current_device())
    n, h, w = int(test_host.shape[0]), int(test_host.shape[1]), int(test_host.shape[2])
    shape = (n, (h * w + 7) // 8) if packed else (n, h, w)
    if out_host is None:
        out_host = t.empty(shape, dtype=t.uint8, pin_memory=True)
    main = t.cuda.current_stream()
    up = up if up is not None else t.cuda.Stream()
    down = t.cuda.Stream()
    # test chunks: double-buffered device frames / masks
    chunk = max(1, min(chunk, n))
    frames = [t.empty((chunk, h, w, 3), dtype=t.uint8, device=dev) for _ in range(2)]
    mshape = (chunk, (h * w + 7) // 8) if packed else (chunk, h, w)
    masks = [t.empty(mshape, dtype=t.uint8, device=dev) for _ in range(2)]
    landed = [t.cuda.Event() for _ in range(2)]
    computed = [t.cuda.Event() for _ in range(2)]
    drained = [t.cuda.Event() for _ in range(2)]
    consumed = [t.cuda.Event() for _ in range(2)]
    for k, s0 in enumerate(range(0, n, chunk)):
        b, m = k & 1, min(chunk, n - s0)
        with t.cuda.stream(up):
            if k >= 2:
                up.wait_event(consumed[b])          # classify of chunk k-2 has read frames[b]
            frames[b][:m].copy_(test_host[s0:s0 + m], non_blocking=True)
            landed[b].record(up)
        main.wait_event(landed[b])
        if k >= 2:
            main.wait_event(drained[b])             # masks[b] of chunk k-2 copied out
        classify(model, frames[b][:m], out=masks[b][:m], packed=packed)
        consumed[b].record(main)
        computed[b].record(main)
        with t.cuda.stream(down):
            down.wait_event(computed[b])
            out_host[s0:s0 + m].copy_(masks[b][:m], non_blocking=True)
            drained[b].record(down)
    main.wait_stream(down)
    main.wait_stream(up)
    return out_host


def detect_sequence(sequence, config: ModelConfig, out_dir=None, batch: int = 64, chunk: int = 16,
                    threads: int = 0):
    """Directory of PPM frames -> background model + foreground masks (SURVEY.md
    §8(f) row 2: the ingest pipeline around the hot path).

    The first ``config.training_frames`` frames (whole groups) build the model;
    then every frame is classified.  Frames are read by host threads straight
    into pinned buffers (``FrameSequence.load_batch``), batch ``i + 1`` is read
    while batch ``i`` goes through the overlapped H2D / classify / D2H chunks,
    and with ``out_dir`` the masks of batch ``i`` are written as 0/255 PGM
    files (``<frame name>.pgm``) by host threads, also in the background.
    Returns (model, masks) -- masks a (n, h, w) uint8 0/1 host tensor -- or
    (model, None) when writing to ``out_dir``.
    """
    from concurrent.futures import ThreadPoolExecutor
    from pathlib import Path
    from .frame_io import FrameSequence, save_masks
    t = _device.torch()
    seq = sequence if isinstance(sequence, FrameSequence) else FrameSequence.scan(sequence)
    n = len(seq)
    n_train = (min(n, config.training_frames) // config.group_size) * config.group_size
    if n_train == 0:
        raise ValueError(f"need at least {config.group_size} frames for one group, got {n}")
    dev = t.device("cuda", t.cuda.current_device())
    train = seq.load_batch(range(n_train), threads=threads).to(dev, non_blocking=True)
    model = build_background_model_device(train, config)
    out = None if out_dir is not None else t.empty((n, seq.height, seq.width), dtype=t.uint8, pin_memory=True)
    if out_dir is not None:
        Path(out_dir).mkdir(parents=True, exist_ok=True)
    starts = list(range(0, n, batch))
    with ThreadPoolExecutor(max_workers=2) as pool:
        nxt = pool.submit(seq.load_batch, range(starts[0], min(n, starts[0] + batch)), None, True, threads)
        writing = None
        for i, s0 in enumerate(starts):
            frames = nxt.result()
            if i + 1 < len(starts):
                s1 = starts[i + 1]
                nxt = pool.submit(seq.load_batch, range(s1, min(n, s1 + batch)), None, True, threads)
            dst = out[s0:s0 + len(frames)] if out is not None else None
            masks = classify_host(model, frames, out_host=dst, chunk=chunk)
            t.cuda.current_stream().synchronize()
            if out_dir is not None:
                if writing is not None:
                    writing.result()
                paths = [Path(out_dir) / (Path(seq.names[s0 + j]).stem + ".pgm") for j in range(len(frames))]
                writing = pool.submit(save_masks, masks, paths, threads)
        if writing is not None:
            writing.result()
    return model, out
