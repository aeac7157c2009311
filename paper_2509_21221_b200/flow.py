"""Thin Python binding of the C-ABI (include/gwtf.h).  Argument marshalling only: every step of
the hot path runs in libgwtf.so's sm_100a kernels.  PyTorch supplies device memory and streams.

Two modes, mirroring GWTF_HOST_PTRS:
  * device (default): inputs/outputs are CUDA torch tensors on the handle's device; calls are
    asynchronous on the stream;
  * host: inputs/outputs are host (ideally pinned) torch tensors; the library copies.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check, lib

ABSENT = 2**31 - 1


def _ptr(t):
    return None if t is None else t.data_ptr()


def _need(t, dtype, shape, name, device):
    if t is None:
        raise ValueError(f"{name} is required")
    if t.dtype != dtype or tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected {dtype} {tuple(shape)}, got {t.dtype} {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device is None:
        if t.is_cuda:
            raise ValueError(f"{name} must be a host tensor on a host-pointer handle")
    elif t.device != device:
        raise ValueError(f"{name} must live on {device}")
    return t


def eq1_cost_tiles(comp, loc, dloc, lat, bw, size_kbit: int, stream=None):
    """Eq. 1 on the device in integer half-units -> (src[B][n], snk[B][n],
    link[B][S-1][n][n]).  All inputs int32 CUDA tensors."""
    B, S, n = comp.shape
    L = lat.shape[1]
    dev = comp.device
    src = torch.empty((B, n), dtype=torch.int32, device=dev)
    snk = torch.empty((B, n), dtype=torch.int32, device=dev)
    link = torch.empty((B, max(S - 1, 0), n, n), dtype=torch.int32, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    check("gwtf_eq1_cost_tiles", lib().gwtf_eq1_cost_tiles(
        B, S, n, L, _ptr(comp), _ptr(loc), _ptr(dloc), _ptr(lat), _ptr(bw), int(size_kbit),
        _ptr(src), _ptr(snk), _ptr(link) if link.numel() else None, st.cuda_stream))
    return src, snk, link


@dataclass
class SolveResult:
    flow_value: torch.Tensor
    total_cost: torch.Tensor
    augmentations: torch.Tensor
    status: torch.Tensor


@dataclass
class RoundsResult:
    rounds_run: torch.Tensor
    dec_flow: torch.Tensor
    dec_cost: torch.Tensor
    dangling: torch.Tensor
    digests: torch.Tensor | None


class Flow:
    """A batch of B routing instances living on one device (gwtf_flow_t)."""

    def __init__(self, cap, src_cost, snk_cost, link_cost, supply, *, max_cap, alive=None, seed=0, inst_base=0,
                 T0=1.7, alpha=0.95, objective=_lib.OBJ_SUM, steady_window=5, deny_after=3, stream=None,
                 host=False, force_global_tier=False, force_cluster_tier=False, warm_repair_all=False):
        B, S, n = cap.shape
        self.B, self.S, self.n, self.max_cap = B, S, n, max_cap
        self.host = host
        if host:
            self.device = torch.device("cuda", torch.cuda.current_device())
            dev_check = None
        else:
            self.device = cap.device
            dev_check = cap.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        _need(cap, torch.int32, (B, S, n), "cap", dev_check)
        _need(src_cost, torch.int32, (B, n), "src_cost", dev_check)
        _need(snk_cost, torch.int32, (B, n), "snk_cost", dev_check)
        if S > 1:
            _need(link_cost, torch.int32, (B, S - 1, n, n), "link_cost", dev_check)
        _need(supply, torch.int64, (B,), "supply", dev_check)
        if alive is not None:
            _need(alive, torch.uint8, (B, S, n), "alive", dev_check)
        self.Mmax = max(1, int(supply.max().item())) if B else 1
        d = _lib.ProblemDesc()
        d.abi_version = _lib.GWTF_ABI_VERSION
        d.num_instances, d.num_stages, d.clients_per_stage, d.max_cap = B, S, n, max_cap
        d.cap, d.alive, d.src_cost, d.snk_cost = _ptr(cap), _ptr(alive), _ptr(src_cost), _ptr(snk_cost)
        d.link_cost = _ptr(link_cost) if S > 1 else None
        d.supply = _ptr(supply)
        d.seed, d.inst_base, d.T0, d.alpha = seed, inst_base, T0, alpha
        d.objective, d.steady_window, d.deny_after = objective, steady_window, deny_after
        d.device = self.device.index if self.device.index is not None else torch.cuda.current_device()
        d.stream = self.stream.cuda_stream
        d.flags = ((_lib.GWTF_HOST_PTRS if host else 0) | (_lib.GWTF_FORCE_GLOBAL_TIER if force_global_tier else 0)
                   | (_lib.GWTF_FORCE_CLUSTER_TIER if force_cluster_tier else 0)
                   | (_lib.GWTF_WARM_REPAIR_ALL if warm_repair_all else 0))
        h = ctypes.c_void_p()
        check("gwtf_flow_create", lib().gwtf_flow_create(ctypes.byref(d), ctypes.byref(h)))
        self.h = h

    # -- helpers
    def _out(self, shape, dtype):
        if self.host:
            return torch.empty(shape, dtype=dtype, pin_memory=True)
        return torch.empty(shape, dtype=dtype, device=self.device)

    def close(self):
        if getattr(self, "h", None):
            lib().gwtf_flow_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- API
    def solve_batch(self, out: SolveResult | None = None) -> SolveResult:
        B = self.B
        if out is None:
            out = SolveResult(self._out((B,), torch.int64), self._out((B,), torch.int64),
                              self._out((B,), torch.int32), self._out((B,), torch.int32))
        check("gwtf_flow_solve_batch", lib().gwtf_flow_solve_batch(
            self.h, _ptr(out.flow_value), _ptr(out.total_cost), _ptr(out.augmentations), _ptr(out.status)))
        return out

    def decentralized_rounds(self, max_rounds: int, digests: bool = False, out: RoundsResult | None = None):
        B = self.B
        if out is None:
            out = RoundsResult(self._out((B,), torch.int32), self._out((B,), torch.int64),
                               self._out((B,), torch.int64), self._out((B,), torch.int32),
                               self._out((B, max(max_rounds, 1)), torch.int64) if digests else None)
        check("gwtf_flow_decentralized_rounds", lib().gwtf_flow_decentralized_rounds(
            self.h, max_rounds, _ptr(out.rounds_run), _ptr(out.dec_flow), _ptr(out.dec_cost), _ptr(out.dangling),
            _ptr(out.digests)))
        return out

    def solve_and_rounds(self, max_rounds: int, out_sol: SolveResult | None = None,
                         out_rounds: RoundsResult | None = None):
        """solve_batch and decentralized_rounds of one step issued together: the rounds run on a
        second stream concurrently with the exact solve (gwtf_flow_solve_and_rounds)."""
        B = self.B
        if out_sol is None:
            out_sol = SolveResult(self._out((B,), torch.int64), self._out((B,), torch.int64),
                                  self._out((B,), torch.int32), self._out((B,), torch.int32))
        if out_rounds is None:
            out_rounds = RoundsResult(self._out((B,), torch.int32), self._out((B,), torch.int64),
                                      self._out((B,), torch.int64), self._out((B,), torch.int32), None)
        check("gwtf_flow_solve_and_rounds", lib().gwtf_flow_solve_and_rounds(
            self.h, max_rounds, _ptr(out_sol.flow_value), _ptr(out_sol.total_cost), _ptr(out_sol.augmentations),
            _ptr(out_sol.status), _ptr(out_rounds.rounds_run), _ptr(out_rounds.dec_flow), _ptr(out_rounds.dec_cost),
            _ptr(out_rounds.dangling)))
        return out_sol, out_rounds

    def _dev(self):
        return None if self.host else self.device

    def apply_churn(self, alive_new=None, edge_updates=None):
        B, S, n = self.B, self.S, self.n
        if alive_new is not None:
            _need(alive_new, torch.uint8, (B, S, n), "alive_new", self._dev())
        k = 0 if edge_updates is None else int(edge_updates.shape[0])
        if edge_updates is not None:
            _need(edge_updates, torch.int32, (k, 5), "edge_updates", self._dev())
        check("gwtf_flow_apply_churn", lib().gwtf_flow_apply_churn(
            self.h, _ptr(alive_new), _ptr(edge_updates) if k else None, k))

    def residual_caps(self):
        """(alive ? cap : 0) - node flow of the last solve (gwtf_flow_residual_caps), [B][S][n] int32."""
        out = self._out((self.B, self.S, self.n), torch.int32)
        check("gwtf_flow_residual_caps", lib().gwtf_flow_residual_caps(self.h, _ptr(out)))
        return out

    def get_assignment(self, dense_arcs: bool = True):
        B, S, n = self.B, self.S, self.n
        nf = self._out((B, S, n), torch.int32)
        sf = self._out((B, n), torch.int32)
        kf = self._out((B, n), torch.int32)
        af = self._out((B, max(S - 1, 0), n, n), torch.int32) if dense_arcs else None
        check("gwtf_flow_get_assignment", lib().gwtf_flow_get_assignment(
            self.h, _ptr(nf), _ptr(sf), _ptr(kf), _ptr(af) if af is not None and af.numel() else None))
        return nf, sf, kf, af

    def export_round_state(self):
        B, S, n, MC, M = self.B, self.S, self.n, self.max_cap, self.Mmax
        st = dict(up=self._out((B, S, n, MC), torch.int32), down=self._out((B, S, n, MC), torch.int32),
                  src_down=self._out((B, M), torch.int32), snk_up=self._out((B, M), torch.int32),
                  kacc=self._out((B, S, n), torch.int32), deny=self._out((B, S, n), torch.int32),
                  quiet=self._out((B,), torch.int32), round=self._out((B,), torch.int64))
        check("gwtf_flow_export_round_state", lib().gwtf_flow_export_round_state(
            self.h, *[_ptr(st[k]) for k in ("up", "down", "src_down", "snk_up", "kacc", "deny", "quiet", "round")]))
        return st

    def import_round_state(self, st: dict):
        """Install a round state in export_round_state()'s layouts (gwtf_flow_import_round_state:
        checkpoint / resume; checked on the device, GwtfError E_INVALID if it is not a valid pairing)."""
        B, S, n, MC, M = self.B, self.S, self.n, self.max_cap, self.Mmax
        shapes = dict(up=(B, S, n, MC), down=(B, S, n, MC), src_down=(B, M), snk_up=(B, M), kacc=(B, S, n),
                      deny=(B, S, n), quiet=(B,), round=(B,))
        args = []
        for key, shape in shapes.items():
            t = st.get(key)
            if t is None and key in ("kacc", "deny", "quiet", "round"):
                args.append(None)
                continue
            args.append(_ptr(_need(t, torch.int64 if key == "round" else torch.int32, shape, key, self._dev())))
        check("gwtf_flow_import_round_state", lib().gwtf_flow_import_round_state(self.h, *args))

    def snapshot(self):
        check("gwtf_flow_snapshot", lib().gwtf_flow_snapshot(self.h))

    def restore(self):
        check("gwtf_flow_restore", lib().gwtf_flow_restore(self.h))

    def set_profiling(self, on: bool):
        check("gwtf_flow_set_profiling", lib().gwtf_flow_set_profiling(self.h, 1 if on else 0))

    def kernel_times(self) -> dict:
        cap = 16
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_float * cap)()
        nl = (ctypes.c_int32 * cap)()
        cnt = ctypes.c_int32()
        check("gwtf_flow_kernel_times", lib().gwtf_flow_kernel_times(
            self.h, names, ctypes.cast(ms, ctypes.c_void_p), ctypes.cast(nl, ctypes.c_void_p), cap,
            ctypes.cast(ctypes.byref(cnt), ctypes.c_void_p)))
        return {names[i].decode(): (ms[i], nl[i]) for i in range(min(cnt.value, cap))}

    def greedy_baseline(self):
        """SWARM-style greedy routing on the current graph (gwtf_flow_greedy_baseline): (routed
        microbatches [B], their total cost [B])."""
        F = self._out((self.B,), torch.int64)
        C = self._out((self.B,), torch.int64)
        check("gwtf_flow_greedy_baseline", lib().gwtf_flow_greedy_baseline(self.h, _ptr(F), _ptr(C)))
        return F, C

    def warm_reroute(self, node_flow, src_flow, snk_flow, arc_flow):
        """Warm-start rerouting on the current (churned) graph from a pre-churn assignment
        (gwtf_flow_warm_reroute).  The four flow tensors (get_assignment's
        layouts, on this handle's side: device or host) are overwritten with the repaired optimum.
        -> (F [B], cost [B], stats [B][3] = stripped / cycles / augmentations, status [B])."""
        B, S, n = self.B, self.S, self.n
        _need(node_flow, torch.int32, (B, S, n), "node_flow", self._dev())
        _need(src_flow, torch.int32, (B, n), "src_flow", self._dev())
        _need(snk_flow, torch.int32, (B, n), "snk_flow", self._dev())
        if arc_flow is not None and arc_flow.numel():
            _need(arc_flow, torch.int32, (B, S - 1, n, n), "arc_flow", self._dev())
        F = self._out((self.B,), torch.int64)
        C = self._out((self.B,), torch.int64)
        St = self._out((self.B, 3), torch.int64)
        Q = self._out((self.B,), torch.int32)
        af = arc_flow if arc_flow is not None and arc_flow.numel() else None
        check("gwtf_flow_warm_reroute", lib().gwtf_flow_warm_reroute(
            self.h, _ptr(node_flow), _ptr(src_flow), _ptr(snk_flow), _ptr(af), _ptr(F), _ptr(C), _ptr(St), _ptr(Q)))
        return F, C, St, Q

    def stats(self, raw: bool = False):
        """Exact-solve work counters since create (gwtf_flow_stats)."""
        import numpy as np
        out = np.zeros(2048, np.int64)
        check("gwtf_flow_stats", lib().gwtf_flow_stats(self.h, out.ctypes.data, 2048))
        if raw:
            return out
        keys = ("relax_steps", "backward_phases", "augmentations", "bf_passes", "path_nodes")
        d = {k: int(out[i]) for i, k in enumerate(keys)}
        d["warm_cold_instances"] = int(out[12])  # instances warm_reroute left to the cold solve
        d["redo_64bit"] = int(out[13])  # instances whose 32-bit keys overflowed (re-solved, 64-bit)
        d["launches"] = int(out[15])
        return d
