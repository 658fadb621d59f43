"""Device-resident batched replay: packed traces that live in HBM.

`DeviceBatch` owns the device copies of a packed batch (requests, offsets,
configs, processing order) plus the engine workspace, and launches
pm_replay_batch on a CUDA stream with no host synchronisation -- the shape a
sweep driver uses when the same traces are replayed many times (config
sweeps, capacity bisection, benchmarking).  PyTorch is only the device
allocator and stream provider here; the kernels are the engine's own.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._native import CFG_DTYPE, REQ_DTYPE, RESULT_DTYPE


def lpt_order(offsets: np.ndarray) -> np.ndarray:
    """Longest trace first, so the persistent warps finish together."""
    lens = np.diff(offsets)
    return np.argsort(-lens, kind="stable").astype(np.int32)


class DeviceBatch:
    def __init__(self, reqs: np.ndarray, offsets: np.ndarray, cfgs: np.ndarray,
                 cfg_of: np.ndarray | None = None, device: int = 0,
                 timeline: bool = False, order: np.ndarray | None = None):
        import torch

        _native.require_device()
        self.lib = _native.load_library()
        self.torch = torch
        self.device = torch.device("cuda", device)
        on_device = isinstance(reqs, torch.Tensor)  # pm_req_t bytes already in HBM
        if not on_device:
            reqs = np.ascontiguousarray(reqs, dtype=REQ_DTYPE)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        cfgs = np.ascontiguousarray(cfgs, dtype=CFG_DTYPE)
        self.n_traces = len(offsets) - 1
        self.total_events = int(offsets[-1] - offsets[0])
        self.max_trace_events = int(np.diff(offsets).max()) if self.n_traces else 0
        if order is None:
            order = lpt_order(offsets)

        def dev(a: np.ndarray):
            t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8))
            return t.to(self.device)

        self.d_reqs = reqs if on_device else dev(reqs)
        self.d_offsets = dev(offsets)
        self.d_cfgs = dev(cfgs)
        self.d_cfg_of = dev(np.ascontiguousarray(cfg_of, dtype=np.int32)) \
            if cfg_of is not None else None
        self.d_order = dev(np.ascontiguousarray(order, dtype=np.int32))
        self.d_results = torch.zeros(self.n_traces * RESULT_DTYPE.itemsize,
                                     dtype=torch.uint8, device=self.device)
        self.d_timeline = (torch.zeros(16 * max(self.total_events, 1),
                                       dtype=torch.uint8, device=self.device)
                           if timeline else None)
        self.ws_bytes = _native.workspace_bytes(
            self.total_events, self.max_trace_events, self.n_traces)
        self.d_ws = torch.empty(self.ws_bytes, dtype=torch.uint8,
                                device=self.device)

    @staticmethod
    def _ptr(t):
        return ctypes.c_void_p(None if t is None else t.data_ptr())

    def launch(self, stream=None) -> None:
        """Enqueue one replay of the whole batch (asynchronous)."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _native.check(self.lib.pm_replay_batch(
            self._ptr(self.d_reqs), self._ptr(self.d_offsets), self.n_traces,
            self._ptr(self.d_cfgs), self._ptr(self.d_cfg_of),
            self._ptr(self.d_order), self._ptr(self.d_results),
            self._ptr(self.d_timeline), self._ptr(self.d_ws), self.ws_bytes,
            self.total_events, self.max_trace_events,
            ctypes.c_void_p(s.cuda_stream)), self.lib)

    def tier_counts(self) -> list[int]:
        """Traces the last launch handed to each retry pass (diagnostic: the
        workspace's control block, csrc/replay_device.cuh Ctl): narrow
        memory-directory passes 1-3, then wide tiers 1-4."""
        ctl = self.d_ws[:64].cpu().numpy().view(np.uint32)
        return [int(x) for x in ctl[9:16]]

    def results(self) -> np.ndarray:
        self.torch.cuda.synchronize(self.device)
        return self.d_results.cpu().numpy().view(RESULT_DTYPE).copy()

    def timeline(self) -> np.ndarray:
        self.torch.cuda.synchronize(self.device)
        return self.d_timeline.cpu().numpy().view(np.int64).copy()

    def capacity_search(self, max_probes: int = 64, stream=None) -> dict:
        """Bisect every trace's smallest runnable device capacity
        (pm_capacity_search; synchronises once per bisection round).

        Returns numpy arrays: min_capacity (n), n_probes (n), unbounded
        (n results), probe_capacity / probe_results ([max_probes, n])."""
        torch = self.torch
        lib = self.lib
        n = self.n_traces
        out = ctypes.c_size_t(0)
        _native.check(lib.pm_capacity_workspace_bytes(
            self.total_events, self.max_trace_events, n, ctypes.byref(out)), lib)
        ws = torch.empty(int(out.value), dtype=torch.uint8, device=self.device)
        dev = self.device
        d_min = torch.zeros(n, dtype=torch.int64, device=dev)
        d_np = torch.zeros(n, dtype=torch.int32, device=dev)
        d_unb = torch.zeros(n * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        d_pcap = torch.full((max_probes * n,), -1, dtype=torch.int64, device=dev)
        d_pres = torch.zeros(max_probes * n * RESULT_DTYPE.itemsize,
                             dtype=torch.uint8, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        _native.check(lib.pm_capacity_search(
            self._ptr(self.d_reqs), self._ptr(self.d_offsets), n,
            self._ptr(self.d_cfgs), self._ptr(self.d_cfg_of),
            self._ptr(self.d_order), self._ptr(d_min), self._ptr(d_np),
            self._ptr(d_unb), self._ptr(d_pcap), self._ptr(d_pres), max_probes,
            self._ptr(ws), int(out.value), self.total_events,
            self.max_trace_events, ctypes.c_void_p(s.cuda_stream)), lib)
        torch.cuda.synchronize(dev)
        return {
            "min_capacity": d_min.cpu().numpy(),
            "n_probes": d_np.cpu().numpy(),
            "unbounded": d_unb.cpu().numpy().view(RESULT_DTYPE).copy(),
            "probe_capacity": d_pcap.cpu().numpy().reshape(max_probes, n),
            "probe_results": d_pres.cpu().numpy().view(RESULT_DTYPE)
                                   .reshape(max_probes, n).copy(),
        }
