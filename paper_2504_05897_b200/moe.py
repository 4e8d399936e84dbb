"""The real HybriMoE MoE layer stack on one B200 (``MoELayer.forward`` of SURVEY.md §8b).

``HybridMoE`` owns one native runtime (include/hybrimoe.h ``hm_runtime_*``):
an HBM slot pool capped at ``floor(ratio * L * N)`` routed experts (+ the
always-resident shared-expert chunks), a pinned host master store, a copy
stream, and the AVX-512 host worker -- and one native decision engine bound
to this package's ``CacheState`` / ``MrsState`` / ``MakespanEvaluator``.
Each layer the GPU router produces the ``LayerRequest`` (loads, scores), the
decision core plans it exactly as the reference's ``run_pass`` would
(engine.py:288-389), and the runtime executes the plan: cached experts on the
GPU, demand copies on the side stream, CPU experts on the host worker.

Routing inputs come either from the reference's synthetic router
(``tracegen.generate_router_logits``; "trace mode") or from the model's own
gate weights applied to the hidden state ("model mode").
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .caching import MrsState, make_mrs_state
from .core import CacheState, ModelConfig, expert_bytes
from .costs import HardwareProfile
from .engine import EnginePolicy, _NativeEngine, cache_capacity
from .scheduling import MakespanEvaluator


@dataclass(frozen=True)
class Family:
    """Router conventions of a model family (see oracle/moe_ref.py for citations)."""

    renormalize: bool
    shared_gate: bool  # Qwen2: shared expert scaled by sigmoid(x . w_sg)


FAMILIES = {
    "tiny": Family(renormalize=True, shared_gate=False),
    "mixtral": Family(renormalize=True, shared_gate=False),
    "deepseek": Family(renormalize=False, shared_gate=False),
    "qwen2": Family(renormalize=False, shared_gate=True),
}

# SURVEY.md §8 configs (bf16 weights: bytes_per_weight = 2; Qwen2 uses the
# released moe_intermediate_size).
SHAPES = {
    "tiny": ModelConfig(num_layers=4, num_routed=8, num_shared=0, num_activated=2, routed_expert_dims=(256, 256),
                        bytes_per_weight=2),
    "mixtral": ModelConfig(num_layers=32, num_routed=8, num_shared=0, num_activated=2,
                           routed_expert_dims=(4096, 14336), bytes_per_weight=2),
    "deepseek": ModelConfig(num_layers=26, num_routed=64, num_shared=2, num_activated=6,
                            routed_expert_dims=(2048, 1408), shared_expert_dims=(2048, 1408), bytes_per_weight=2),
    "qwen2": ModelConfig(num_layers=28, num_routed=64, num_shared=1, num_activated=8,
                         routed_expert_dims=(3584, 2560), shared_expert_dims=(3584, 20480), bytes_per_weight=2),
}


def shared_chunks(cfg: ModelConfig) -> int:
    """Shared experts as always-resident chunks of the routed shape: SwiGLU is
    separable along the intermediate dimension, so one (H, k*I) shared expert
    is exactly the sum of k (H, I) experts."""
    if not cfg.num_shared or cfg.shared_expert_dims is None:
        return 0
    H, I = cfg.routed_expert_dims
    sh, si = cfg.shared_expert_dims
    if sh != H or si % I:
        raise ValueError(f"shared expert dims {cfg.shared_expert_dims} are not whole chunks of {cfg.routed_expert_dims}")
    return cfg.num_shared * (si // I)


class _Raw:
    """__cuda_array_interface__ / __array_interface__ shim to view native buffers as tensors."""

    def __init__(self, ptr: int, n: int, cuda: bool) -> None:
        typestr = "<i2" if cuda else "<u2"
        iface = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}
        if cuda:
            iface["strides"] = None
            self.__cuda_array_interface__ = iface
        else:
            self.__array_interface__ = iface


class TracePredictor:
    """Trace-mode prediction input for forward_pass: the pass's true loads, fed
    through the reference's noisy-ground-truth model natively (prefetch.py:54-101)."""

    def __init__(self, trace, pass_index: int, seed: int) -> None:
        self.pass_loads = np.ascontiguousarray([r.loads for r in trace.passes[pass_index].layers], dtype=np.int64)
        self.pass_index = int(pass_index)
        self.seed = int(seed)


@dataclass
class LayerStats:
    makespan_planned: float
    t_wait_router_us: float
    t_decide_us: float
    t_cpu_us: float
    n_gpu: int
    n_cpu: int
    n_transfer: int
    n_prefetch: int
    bytes_gpu: int
    bytes_cpu: int
    bytes_h2d: int


def layer_stats(info: dict) -> list[LayerStats]:
    """Per-layer stats of a forward_pass info dict (native passes keep raw structs)."""
    if "stats" in info:
        return info["stats"]
    return [LayerStats(*[getattr(s, f) for f, _ in _lib.LayerStats._fields_]) for s in info["stats_raw"]]


class HybridMoE:
    """L MoE layers (router + experts + combine, residual stream) under the HybriMoE schedule."""

    def __init__(self, config: ModelConfig, family: str, policy: EnginePolicy, capacity_ratio: float,
                 profile: HardwareProfile, *, host_images: int | None = None, max_tokens: int = 1024,
                 cpu_threads: int = 0, gpu_mrs: bool = True, residual: bool = True, ep_rank: int = 0,
                 ep_world: int = 1, process_group=None, exchange: str = "p2p", weight_bits: int = 16) -> None:
        if not torch.cuda.is_available():
            raise RuntimeError("HybridMoE executes on a CUDA device; no CPU fallback exists")
        self.config = config
        self.family = FAMILIES[family]
        self.policy = policy
        self.profile = profile
        H, I = config.routed_expert_dims
        self.H, self.I = H, I
        self.L, self.N, self.K = config.num_layers, config.num_routed, config.num_activated
        self.S = shared_chunks(config)
        self.ep_rank, self.ep_world, self.group = int(ep_rank), max(1, int(ep_world)), process_group
        if self.ep_world > 1:  # this rank's share of the global budget (ep.py)
            from .ep import rank_capacity
            self.capacity = rank_capacity(config, capacity_ratio, self.ep_rank, self.ep_world)
        else:
            self.capacity = cache_capacity(config, capacity_ratio)
        self.cache = CacheState(self.capacity)
        self.mrs: MrsState = make_mrs_state(config, alpha=policy.mrs_alpha, p=policy.mrs_p)
        self.evaluator = MakespanEvaluator(profile, expert_bytes(config))
        split = policy.static_split_point
        if split is None:
            split = math.floor(capacity_ratio * config.num_layers)
        self.engine = _NativeEngine(config, policy, self.cache, self.mrs, self.evaluator, profile, split,
                                    frozenset(), collect=True)
        n_home = (self.N - self.ep_rank + self.ep_world - 1) // self.ep_world
        total = self.L * n_home
        self.host_images = total if host_images is None else max(1, min(int(host_images), total))
        self.gate_col = self.N if self.family.shared_gate else -1
        self.ld = self.N + (1 if self.family.shared_gate else 0)
        rc = _lib.RuntimeConfig(num_layers=self.L, num_routed=self.N, num_activated=self.K, hidden=H, inter=I,
                                n_shared=self.S, renormalize=int(self.family.renormalize),
                                shared_gate_col=self.gate_col, capacity=self.capacity,
                                host_images=self.host_images, cpu_threads=int(cpu_threads),
                                max_tokens=int(max_tokens), gpu_mrs=int(gpu_mrs), residual=int(residual),
                                ep_rank=self.ep_rank, ep_world=self.ep_world, weight_bits=int(weight_bits))
        h = C.c_void_p()
        check(lib.hm_runtime_create(C.byref(rc), self.engine._h, C.byref(h)))
        self._rt = h.value
        self.residual = residual
        self.y32 = None
        self.exchange = exchange if self.ep_world > 1 else "none"
        self._ep = None
        if self.ep_world > 1:
            if exchange == "p2p":  # combine + cross-rank sum in one kernel over peer memory
                from .ep import P2PExchange
                self._ep = P2PExchange(self.ep_rank, self.ep_world, max_tokens, H, process_group)
                check(lib.hm_runtime_set_ep_exchange(self._rt, self._ep.handle))
            elif exchange == "dispatch":  # token-sharded: all-to-all of rows to home ranks and back
                from .ep import P2PExchange
                self._ep = P2PExchange(self.ep_rank, self.ep_world, max_tokens, H, process_group,
                                       dispatch=(self.N + self.S, self.N, self.K + self.S))
                check(lib.hm_runtime_set_ep_dispatch(self._rt, self._ep.handle))
            elif exchange == "nccl_a2a":  # token-sharded over NCCL grouped send/recv (baseline / fallback)
                from .ep import NcclExchange
                self._ep = NcclExchange(self.ep_rank, self.ep_world, max_tokens, H,
                                        (self.N + self.S, self.N, self.K + self.S), process_group)
                check(lib.hm_runtime_set_ep_dispatch(self._rt, self._ep.handle))
            elif exchange == "allreduce":  # baseline: partials all-reduced on the process group
                self.y32 = torch.empty((max_tokens, H), dtype=torch.float32, device="cuda")
                check(lib.hm_runtime_set_ep_output(self._rt, self.y32.data_ptr()))
            else:
                raise ValueError(f"unknown expert-parallel exchange {exchange!r} (p2p | dispatch | nccl_a2a | allreduce)")
        pool, store, sb, ns = C.c_void_p(), C.c_void_p(), C.c_size_t(), C.c_int64()
        check(lib.hm_runtime_buffers(self._rt, C.byref(pool), C.byref(store), C.byref(sb), C.byref(ns)))
        self.slot_bytes, self.n_slots = sb.value, ns.value
        self.slot_elems = self.slot_bytes // 2
        self.pool = (torch.as_tensor(_Raw(pool.value, self.n_slots * self.slot_elems, True), device="cuda")
                     .view(torch.bfloat16).view(self.n_slots, self.slot_elems) if self.n_slots else None)
        self.store = np.asarray(_Raw(store.value, self.host_images * self.slot_elems, False)).reshape(
            self.host_images, self.slot_elems)
        self.store_t = torch.from_numpy(self.store.view(np.int16)).view(torch.bfloat16)
        self.weight_bits = int(weight_bits)
        self.image_bytes = 3 * H * I * 2
        if self.weight_bits == 4:  # 4-bit images: bytes of one image inside its (aligned) slot
            nb = C.c_size_t()
            check(lib.hm_q4_image_bytes(H, I, C.byref(nb)))
            self.image_bytes = nb.value
        self.gate_w: torch.Tensor | None = None
        self.max_tokens = max_tokens
        self._bufs: dict[int, tuple[torch.Tensor, torch.Tensor]] = {}
        # fixed residency of the baseline schedulings: static_layer_split keeps
        # the layers below the split on the GPU (engine.py:185-192); those
        # experts (this rank's home share) are copied into slots once weights exist
        self._fixed_refs: list[tuple[int, int]] = []
        self._weights_ready = False
        if policy.scheduling == "static_layer_split":
            refs = [(l, e) for l in range(split) for e in range(self.N) if e % self.ep_world == self.ep_rank]
            if len(refs) > self.capacity:
                raise ValueError(f"static_layer_split keeps {len(refs)} experts of layers < {split} on this GPU, "
                                 f"more than its {self.capacity} cache slots")
            self._fixed_refs = refs

    def close(self) -> None:
        """Release the runtime now (HBM slot pool, pinned master store, host
        worker threads) whatever still references this object; idempotent."""
        if getattr(self, "_rt", None):
            torch.cuda.synchronize()
            lib.hm_runtime_destroy(self._rt)
            self._rt = None
        if getattr(self, "_ep", None) is not None:
            self._ep.close()
            self._ep = None

    def __del__(self) -> None:
        self.close()

    # -------------------------------------------------------------- weights
    def _encode(self, bf16_images: torch.Tensor) -> torch.Tensor:
        """bf16 expert images [k, 3HI] (device) -> slot contents [k, slot_elems]
        (bf16 view): the images themselves, or their 4-bit quantization."""
        if self.weight_bits != 4:
            return bf16_images
        k = bf16_images.shape[0]
        q = torch.zeros((k, self.slot_bytes), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        for i in range(k):
            check(lib.hm_q4_quantize(bf16_images[i].data_ptr(), self.H, self.I, q[i].data_ptr(), st))
        return q.view(torch.bfloat16)

    def init_random_weights(self, seed: int = 0, chunk_images: int = 8) -> None:
        """Random-init N(0, 0.02^2) bf16 experts, generated on the
        GPU (4-bit runs quantize them there) and written to the pinned master
        store / shared slots; router gate weights N(0, 1/H) for model mode."""
        g = torch.Generator(device="cuda").manual_seed(seed)
        n = 3 * self.H * self.I
        for i0 in range(0, self.host_images, chunk_images):
            k = min(chunk_images, self.host_images - i0)
            buf = (torch.randn((k, n), generator=g, device="cuda", dtype=torch.float32) * 0.02).to(torch.bfloat16)
            self.store_t[i0:i0 + k].copy_(self._encode(buf))
        for l in range(self.L):
            for c in range(self.S):
                s = self.shared_slot(l, c)
                self.pool[s].copy_(self._encode((torch.randn((1, n), generator=g, device="cuda") * 0.02).to(
                    torch.bfloat16))[0])
        self.gate_w = (torch.randn((self.L, self.ld, self.H), generator=g, device="cuda") / math.sqrt(self.H)).to(
            torch.bfloat16)
        torch.cuda.synchronize()
        self._weights_ready = True
        self._apply_residency()

    def init_seeded_weights(self, base_seed: int = 0) -> None:
        """Per-expert seeded init (torch.Generator seed 1000*layer +
        expert): the same expert gets the same weights on any rank count, so an
        expert-parallel run can be compared with a single-GPU one."""
        n = 3 * self.H * self.I
        for l in range(self.L):
            for e in range(self.N):
                if e % self.ep_world != self.ep_rank:
                    continue
                g = torch.Generator(device="cuda").manual_seed(base_seed + 1000 * l + e)
                self.store_t[self.image_of(l, e)].copy_(self._encode(
                    (torch.randn((1, n), generator=g, device="cuda") * 0.02).to(torch.bfloat16))[0])
            for c in range(self.S):
                g = torch.Generator(device="cuda").manual_seed(base_seed + 1000 * l + self.N + c)
                self.pool[self.shared_slot(l, c)].copy_(self._encode(
                    (torch.randn((1, n), generator=g, device="cuda") * 0.02).to(torch.bfloat16))[0])
        g = torch.Generator(device="cuda").manual_seed(base_seed + 999_999)
        self.gate_w = (torch.randn((self.L, self.ld, self.H), generator=g, device="cuda") / math.sqrt(self.H)).to(
            torch.bfloat16)
        torch.cuda.synchronize()
        self._weights_ready = True
        self._apply_residency()

    # checkpoint loading (e.g. a transformers MoE block's parameters); call
    # before the first forward pass -- resident HBM copies are not refreshed
    def _image(self, gate: torch.Tensor, up: torch.Tensor, down: torch.Tensor) -> torch.Tensor:
        """gate/up [I, H], down [H, I] -> one bf16 slot image [1, 3HI] on the GPU
        (W13 rows interleaved in 128-row gate/up blocks, include/hybrimoe.h)."""
        H, I = self.H, self.I
        if tuple(gate.shape) != (I, H) or tuple(up.shape) != (I, H) or tuple(down.shape) != (H, I):
            raise ValueError(f"expert weights must be gate/up [{I}, {H}] and down [{H}, {I}]")
        g = gate.to("cuda", torch.bfloat16).reshape(I // 128, 1, 128, H)
        u = up.to("cuda", torch.bfloat16).reshape(I // 128, 1, 128, H)
        w13 = torch.cat([g, u], dim=1).reshape(-1)
        return torch.cat([w13, down.to("cuda", torch.bfloat16).reshape(-1)]).reshape(1, -1)

    def set_expert_weights(self, layer: int, expert: int, gate: torch.Tensor, up: torch.Tensor,
                           down: torch.Tensor) -> None:
        """Routed expert (layer, expert) into the pinned master store (ignored
        on a rank that is not the expert's home)."""
        if expert % self.ep_world != self.ep_rank:
            return
        n_home = (self.N - self.ep_rank + self.ep_world - 1) // self.ep_world
        if self.host_images < self.L * n_home:
            raise ValueError("per-expert weights need one host image per expert (host_images aliases them)")
        self.store_t[self.image_of(layer, expert)].copy_(self._encode(self._image(gate, up, down))[0])
        self._weights_ready = True

    def set_shared_weights(self, layer: int, gate: torch.Tensor, up: torch.Tensor, down: torch.Tensor) -> None:
        """The layer's shared expert(s) as ONE SwiGLU of intermediate size
        S*I (gate/up [S*I, H], down [H, S*I]: DeepSeek's n_shared experts
        concatenated, Qwen2's single wide one), split into its S resident chunks."""
        I = self.I
        if gate.shape[0] != self.S * I:
            raise ValueError(f"shared expert intermediate size {gate.shape[0]} != {self.S} chunks x {I}")
        for c in range(self.S):
            sl = slice(c * I, (c + 1) * I)
            self.pool[self.shared_slot(layer, c)].copy_(
                self._encode(self._image(gate[sl], up[sl], down[:, sl]))[0])

    def set_router_weights(self, layer: int, weight: torch.Tensor, shared_gate: torch.Tensor | None = None) -> None:
        """Router gate [N, H] (and the Qwen2 shared-expert gate [1, H]) of a layer,
        for model mode (logits computed on the GPU from the hidden state)."""
        if self.gate_w is None:
            self.gate_w = torch.zeros((self.L, self.ld, self.H), dtype=torch.bfloat16, device="cuda")
        self.gate_w[layer, : self.N] = weight.to("cuda", torch.bfloat16)
        if self.family.shared_gate:
            if shared_gate is None:
                raise ValueError("this family's router needs the shared-expert gate row")
            self.gate_w[layer, self.N] = shared_gate.reshape(-1).to("cuda", torch.bfloat16)

    def _apply_residency(self) -> None:
        """(Re)copy the fixed-residency experts into their slots (after weights change)."""
        if self._fixed_refs and self._weights_ready:
            self.preload(self._fixed_refs)

    def set_profile(self, profile: HardwareProfile) -> None:
        """Plan the following passes with another calibrated profile (e.g. the
        prefill profile for the prefill pass, the decode profile after it)."""
        from .costs import to_native
        self.profile = profile
        self.evaluator.profile = profile
        check(lib.hm_engine_set_profile(self.engine._h, C.byref(to_native(profile))))

    def preload(self, refs) -> None:
        """Fixed residency for the baseline schedulings (engine.py:423-434):
        make these experts resident and copy them into their HBM slots."""
        refs = list(refs)
        arr = (C.c_uint32 * max(1, len(refs)))(*[(int(l) << 16) | int(e) for l, e in refs])
        check(lib.hm_runtime_preload(self._rt, arr, len(refs)))

    def set_fixed_gpu_set(self, refs) -> None:
        """fixed_frequency_map's GPU-pinned set (engine.py:195-231), made resident."""
        refs = [(int(l), int(e)) for l, e in refs]
        if len(refs) > self.capacity:
            raise ValueError(f"fixed GPU set of {len(refs)} experts exceeds the {self.capacity} cache slots")
        arr = (C.c_uint32 * max(1, len(refs)))(*[(l << 16) | e for l, e in refs])
        check(lib.hm_engine_set_fixed_pinned(self.engine._h, arr, len(refs)))
        self._fixed_refs = refs
        self._apply_residency()

    def image_of(self, layer: int, expert: int) -> int:
        v = C.c_int64()
        check(lib.hm_runtime_image_of(self._rt, layer, expert, C.byref(v)))
        return v.value

    def shared_slot(self, layer: int, chunk: int) -> int:
        v = C.c_int64()
        check(lib.hm_runtime_shared_slot(self._rt, layer, chunk, C.byref(v)))
        return v.value

    def expert_image(self, layer: int, expert: int) -> np.ndarray:
        """Host bytes of routed expert (layer, expert) in slot layout (uint16 bf16
        bits; for 4-bit runs the uint8 bytes of the 4-bit image)."""
        img = self.store[self.image_of(layer, expert)]
        return img.view(np.uint8)[: self.image_bytes] if self.weight_bits == 4 else img

    def shared_image(self, layer: int, chunk: int) -> np.ndarray:
        img = self.pool[self.shared_slot(layer, chunk)].view(torch.int16).cpu().numpy().view(np.uint16)
        return img.view(np.uint8)[: self.image_bytes] if self.weight_bits == 4 else img

    # -------------------------------------------------------------- forward
    def _ping_pong(self, T: int) -> tuple[torch.Tensor, torch.Tensor]:
        if T not in self._bufs:
            self._bufs[T] = tuple(torch.empty((T, self.H), dtype=torch.bfloat16, device="cuda") for _ in range(2))
        return self._bufs[T]

    def forward_pass(self, x: torch.Tensor, logits=None, predict=None, decision_log: bool = False,
                     keep_layers: bool = False, stream=None):
        """Run all L layers on x [T, H] bf16.

        logits: per-layer [T, ld] fp32 CUDA tensors (trace mode) or None (model
        mode: x_l . W_g,l).  predict(layer) -> list of predicted LayerRequests
        for the prefetch decision (prefetch.py:54-101).  Returns (y, info)."""
        if not getattr(self, "_rt", None):
            raise RuntimeError("this HybridMoE was closed")
        T = x.shape[0]
        if T > self.max_tokens:
            raise ValueError(f"T={T} exceeds max_tokens={self.max_tokens}")
        st = stream if stream is not None else torch.cuda.current_stream()
        a, b = self._ping_pong(T)
        live = predict == "live" and self.policy.prefetch
        if live:
            self._set_lookahead()
        if ((self.ep_world == 1 or self._ep is not None) and logits is not None and not decision_log and not keep_layers
                and (predict is None or isinstance(predict, TracePredictor) or live or not self.policy.prefetch)):
            return self._forward_pass_native(x, logits, predict, a, b, st)
        cur = x
        stats, records, layers_io, requests = [], [], [], []
        ls = _lib.LayerStats()
        loads = np.zeros(self.N, dtype=np.int64)
        scores = np.zeros(self.N, dtype=np.float64)
        self.engine.begin_pass()
        hz = self.policy.prediction.horizon
        npred = C.c_int()
        for l in range(self.L):
            lg = logits[l] if logits is not None else self._model_logits(cur, l, st)
            if self.policy.prefetch and isinstance(predict, TracePredictor):
                # the reference's prediction model, natively (csrc/predict.cpp)
                pl = np.empty(hz, dtype=np.int32)
                pload = np.empty((hz, self.N), dtype=np.int64)
                check(lib.hm_predict_layers(_lib.ptr(predict.pass_loads, C.c_int64), self.L, self.N,
                                            predict.pass_index, l, predict.seed, hz,
                                            float(self.policy.prediction.accuracy), _lib.ptr(pl, C.c_int32),
                                            _lib.ptr(pload, C.c_int64), C.byref(npred)))
                pl = pl[: npred.value]
            elif live:  # native look-ahead, launched ahead of this layer's router
                pl, pload = np.zeros(1, np.int32), np.zeros((1, self.N), np.int64)
            else:
                if not self.policy.prefetch:
                    preds = []
                elif predict == "live_py":  # the same look-ahead through the Python kernels (checker)
                    preds = self.lookahead(cur, l, stream=st)
                else:
                    preds = predict(l) if predict is not None else []
                pl = np.array([p.layer for p in preds], dtype=np.int32)
                pload = np.zeros((max(1, len(preds)), self.N), dtype=np.int64)
                for d, p in enumerate(preds):
                    for i in p.activated:
                        pload[d, i] = p.loads[i]
            out = a if (l % 2 == 0) else b
            check(lib.hm_runtime_forward_layer(self._rt, l, cur.data_ptr(), lg.data_ptr(), T, lg.shape[1],
                                               out.data_ptr(), _lib.ptr(pl, C.c_int32), _lib.ptr(pload, C.c_int64),
                                               _lib.HM_PREDICT_LIVE if live else len(pl), st.cuda_stream,
                                               C.byref(ls)))
            if self.ep_world > 1 and self._ep is None:  # all-reduce the ranks' partials, then the residual
                import torch.distributed as dist
                part = self.y32[:T]
                with torch.cuda.stream(st):
                    dist.all_reduce(part, group=self.group)
                    if self.residual:
                        check(lib.hm_residual_add(part.data_ptr(), cur.data_ptr(), T, self.H, out.data_ptr(),
                                                  st.cuda_stream))
                    else:  # test configuration: the layer output is the MoE sum alone
                        out.copy_(part.to(torch.bfloat16))
            stats.append(LayerStats(*[getattr(ls, f) for f, _ in _lib.LayerStats._fields_]))
            if decision_log:
                rec = self.engine.record()
                rec["layer"] = l
                rec["mrs_row"] = self.mrs.table()[l].copy()
                records.append(rec)
                check(lib.hm_runtime_last_request(self._rt, _lib.ptr(loads, C.c_int64), _lib.ptr(scores, C.c_double)))
                requests.append((loads.copy(), scores.copy()))
            if keep_layers:  # clones are ordered after this layer on the same stream
                with torch.cuda.stream(st):
                    layers_io.append((cur.clone(), lg, out.clone()))
            cur = out
        r = self.engine.end_pass()
        info = {"stats": stats, "records": records, "requests": requests, "layers": layers_io, "pass": r}
        return cur, info

    def _forward_pass_native(self, x, logits, predict, a, b, st):
        """The whole pass in one native call (hm_runtime_forward_pass): no Python per layer."""
        T = x.shape[0]
        lgp = (C.c_void_p * self.L)(*[lg.data_ptr() for lg in logits])
        stats = (_lib.LayerStats * self.L)()
        res = _lib.PassResult()
        yp = C.c_void_p()
        pl = predict if isinstance(predict, TracePredictor) and self.policy.prefetch else None
        if pl is None and predict != "live":
            self._set_lookahead(off=True)
        check(lib.hm_runtime_forward_pass(
            self._rt, x.data_ptr(), lgp, T, logits[0].shape[1], a.data_ptr(), b.data_ptr(),
            _lib.ptr(pl.pass_loads, C.c_int64) if pl is not None else None, pl.pass_index if pl else 0,
            pl.seed if pl else 0, self.policy.prediction.horizon, float(self.policy.prediction.accuracy),
            st.cuda_stream, stats, C.byref(res), C.byref(yp)))
        y = a if yp.value == a.data_ptr() else b
        return y, {"stats_raw": stats, "records": [], "requests": [], "layers": [], "pass": res}

    def _set_lookahead(self, off: bool = False) -> None:
        """Point the runtime's live predictor at the gate weights (or detach it)."""
        want = None if off or self.gate_w is None else (self.gate_w.data_ptr(), self.policy.prediction.horizon)
        if want is None and not off:
            raise RuntimeError("live prediction needs gate weights (init_random_weights)")
        if getattr(self, "_la", None) != want:
            check(lib.hm_runtime_set_lookahead(self._rt, want[0] if want else None, self.ld, want[1] if want else 0))
            self._la = want

    def lookahead(self, x: torch.Tensor, layer: int, horizon: int | None = None, stream=None):
        """Live-mode prediction: the gates of layers
        l+1..l+H applied to the current hidden state give the predicted
        LayerRequests the prefetch decision evaluates (prefetch.py:104-143)."""
        from .core import LayerRequest
        from .kernels import router_logits, router_topk

        if self.gate_w is None:
            raise RuntimeError("live prediction needs gate weights (init_random_weights)")
        hz = self.policy.prediction.horizon if horizon is None else horizon
        last = min(layer + hz, self.L - 1)
        out = []
        for fl in range(layer + 1, last + 1):
            lg = router_logits(x, self.gate_w[fl], stream=stream)
            _, _, _, counts = router_topk(lg, self.N, self.K, self.family.renormalize, 0, -1, stream=stream)
            loads = counts.cpu().numpy().astype(np.int64)
            out.append(LayerRequest(layer=fl, loads=tuple(int(v) for v in loads), scores=(),
                                    activated=frozenset(int(i) for i in np.nonzero(loads)[0])))
        return out

    def _model_logits(self, x: torch.Tensor, layer: int, st) -> torch.Tensor:
        from .kernels import router_logits
        if self.gate_w is None:
            raise RuntimeError("model mode needs gate weights (init_random_weights)")
        return router_logits(x, self.gate_w[layer], stream=st)

    def device_mrs(self) -> np.ndarray:
        out = np.empty((self.L, self.N), dtype=np.float64)
        check(lib.hm_runtime_device_mrs(self._rt, _lib.ptr(out, C.c_double)))
        return out

    def sync(self) -> None:
        check(lib.hm_runtime_sync(self._rt))
        torch.cuda.synchronize()


def with_shared_time(profile: HardwareProfile, cfg: ModelConfig) -> HardwareProfile:
    """Shared chunks run inside every layer's GPU batch; account them like the
    reference's constant per-layer shared_expert_time (costs.py:44, engine.py:307)."""
    return replace(profile, shared_expert_time=shared_chunks(cfg) * profile.gpu_time_per_expert)
