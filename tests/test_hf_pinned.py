"""Expert numerics pinned to an independent implementation: the MoE blocks of
HuggingFace transformers 5.5 for the three model families the configs name.

The reference simulator never evaluates an expert, so the fp32
oracle (oracle/moe_ref.py) restates Eq. 1 with each family's router.  Here
that restatement is checked against transformers' own modules on the same
bf16-valued weights and inputs --
  Mixtral   MixtralSparseMoeBlock   (softmax -> top-K -> renormalise)
  DeepSeek  DeepseekV2Moe           (softmax -> greedy top-K, x routed_scaling_factor, + shared experts)
  Qwen2-MoE Qwen2MoeSparseMoeBlock  (softmax -> top-K, + sigmoid-gated shared expert)
-- on CPU in fp32 (tolerance 1e-4: summation order only), and the B200 layer
(router + permutation + GEMV / tcgen05 GEMM + combine, weights loaded through
HybridMoE.set_*_weights) against the same modules at the stated bf16
tolerance 1e-2.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import moe_ref as ref

transformers = pytest.importorskip("transformers")

H, I = 256, 256
# the released shapes: (H, I, routed experts, top-K)
FULL = {"mixtral": (4096, 14336, 8, 2), "deepseek": (2048, 1408, 64, 6), "qwen2": (3584, 2560, 64, 8)}


def _block(family: str, seed: int, dims=None, device: str = "cpu"):
    """A transformers MoE block of the family at reduced dims (or `dims` =
    (H, I, N, K)), weights N(0, 0.02) / router N(0, 1/H), all bf16-valued."""
    from transformers import DeepseekV2Config, MixtralConfig, Qwen2MoeConfig
    H_, I_, N_, K_ = dims or (H, I, None, None)
    torch.manual_seed(seed)
    if family == "mixtral":
        from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock
        n, k = N_ or 8, K_ or 2
        cfg = MixtralConfig(hidden_size=H_, intermediate_size=I_, num_local_experts=n, num_experts_per_tok=k)
        cfg._experts_implementation = "eager"
        blk, s_int = MixtralSparseMoeBlock(cfg), 0
    elif family == "deepseek":
        from transformers.models.deepseek_v2.modeling_deepseek_v2 import DeepseekV2Moe
        n, k = N_ or 16, K_ or 6
        cfg = DeepseekV2Config(hidden_size=H_, moe_intermediate_size=I_, n_routed_experts=n, num_experts_per_tok=k,
                               n_shared_experts=2, routed_scaling_factor=1.0, topk_method="greedy", n_group=1,
                               topk_group=1)
        cfg._experts_implementation = "eager"
        blk, s_int = DeepseekV2Moe(cfg), 2 * I_
    else:
        from transformers.models.qwen2_moe.modeling_qwen2_moe import Qwen2MoeSparseMoeBlock
        n, k = N_ or 16, K_ or 4
        cfg = Qwen2MoeConfig(hidden_size=H_, moe_intermediate_size=I_, shared_expert_intermediate_size=8 * I_,
                             num_experts=n, num_experts_per_tok=k, norm_topk_prob=False)
        cfg._experts_implementation = "eager"
        blk, s_int = Qwen2MoeSparseMoeBlock(cfg), 8 * I_
    blk = blk.to(device)
    g = torch.Generator(device=device).manual_seed(seed)
    with torch.no_grad():  # N(0, 0.02) experts, N(0, 1/H) router, every value bf16-representable
        for name, prm in blk.named_parameters():
            std = 1.0 / np.sqrt(H_) if "gate.weight" in name else 0.02
            prm.copy_((torch.randn(prm.shape, generator=g, device=device) * std).to(torch.bfloat16).float())
    return blk.eval(), n, k, s_int


def _params(blk, family: str, n: int):
    """(routed experts [(gate, up, down)], shared (gate, up, down) or None,
    router [N, H], shared gate [1, H] or None) as fp32 tensors."""
    gu, dn = blk.experts.gate_up_proj.detach(), blk.experts.down_proj.detach()
    i_ = dn.shape[2]
    routed = [(gu[e, :i_], gu[e, i_:], dn[e]) for e in range(n)]
    shared, sgate = None, None
    if family == "deepseek":
        m = blk.shared_experts
        shared = (m.gate_proj.weight.detach(), m.up_proj.weight.detach(), m.down_proj.weight.detach())
    elif family == "qwen2":
        m = blk.shared_expert
        shared = (m.gate_proj.weight.detach(), m.up_proj.weight.detach(), m.down_proj.weight.detach())
        sgate = blk.shared_expert_gate.weight.detach()
    return routed, shared, blk.gate.weight.detach(), sgate


def _logits(x: torch.Tensor, router: torch.Tensor, sgate):
    w = router if sgate is None else torch.cat([router, sgate], 0)
    return (x.float().to(w.device) @ w.float().T).cpu().numpy().astype(np.float32)


def _oracle(family, blk, n, k, x):
    routed, shared, router, sgate = _params(blk, family, n)
    experts = [tuple(t.numpy() for t in e) for e in routed]
    n_sh = 0
    if shared is not None:  # the shared SwiGLU as chunks of the routed width (separable along I)
        g, u, d = (t.numpy() for t in shared)
        n_sh = g.shape[0] // I
        experts += [(g[c * I:(c + 1) * I], u[c * I:(c + 1) * I], d[:, c * I:(c + 1) * I]) for c in range(n_sh)]
    return ref.moe_layer(x.numpy(), _logits(x, router, sgate), experts, n, k, family == "mixtral", n_sh,
                         n if sgate is not None else -1)


@pytest.mark.parametrize("family", ["mixtral", "deepseek", "qwen2"])
@pytest.mark.parametrize("T", [1, 16])
def test_oracle_matches_transformers_moe_block(family, T):
    blk, n, k, _ = _block(family, 3 + T)
    x = torch.randn(T, H).to(torch.bfloat16).float()
    with torch.no_grad():
        want = blk(x.reshape(1, T, H)).reshape(T, H).numpy()
    got = _oracle(family, blk, n, k, x)
    assert np.abs(got - want).max() / np.abs(want).max() <= 1e-4


def _hybrid(family, blk, n, k, s_int, T, cpu_slope, H=H, I=I):
    import paper_2504_05897_b200.core as mcore
    import paper_2504_05897_b200.costs as mcost
    import paper_2504_05897_b200.engine as me
    from paper_2504_05897_b200.moe import HybridMoE
    cfg = mcore.ModelConfig(num_layers=1, num_routed=n, num_shared=(2 if family == "deepseek" else 1) if s_int else 0,
                            num_activated=k, routed_expert_dims=(H, I),
                            shared_expert_dims=(H, I if family == "deepseek" else s_int) if s_int else None,
                            bytes_per_weight=2)
    eb = mcore.expert_bytes(cfg)
    prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=cpu_slope, transfer_bandwidth=eb / 0.5)
    # budget = every expert (one layer: a full cache of pinned residents would be
    # the reference's EvictionError, caching.py:111-128)
    moe = HybridMoE(cfg, family, me.EnginePolicy(), 1.0, prof, max_tokens=max(T, 8), residual=False)
    routed, shared, router, sgate = _params(blk, family, n)
    for e, (g, u, d) in enumerate(routed):
        moe.set_expert_weights(0, e, g, u, d)
    if shared is not None:
        moe.set_shared_weights(0, *shared)
    moe.set_router_weights(0, router, sgate)
    return moe, router, sgate


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["mixtral", "deepseek", "qwen2"])
@pytest.mark.parametrize("T", [1, 3, 200])
@pytest.mark.parametrize("placement", ["host", "gpu"])
def test_b200_layer_matches_transformers_moe_block(family, T, placement):
    """GEMV path (T = 1, 3) and tcgen05 GEMM path (T = 200: > 4 rows per
    expert); the profile steers the plan to the host worker (cheap CPU) or to
    transfers + GPU kernels (expensive CPU), and the stats confirm where the
    routed experts ran."""
    from paper_2504_05897_b200.moe import layer_stats
    blk, n, k, s_int = _block(family, 11 + T)
    moe, router, sgate = _hybrid(family, blk, n, k, s_int, T, 1e-3 if placement == "host" else 1e3)
    x = torch.randn(T, H).to(torch.bfloat16)
    with torch.no_grad():
        want = blk(x.float().reshape(1, T, H)).reshape(T, H).numpy()
    lg = torch.from_numpy(_logits(x.float(), router, sgate)).cuda()
    for _ in range(2):  # a cold and a warm pass (cache state differs, plan differs)
        y, info = moe.forward_pass(x.cuda(), [lg])
        torch.cuda.synchronize()
        got = y.float().cpu().numpy()
        assert np.abs(got - want).max() / np.abs(want).max() <= 1e-2
        st = layer_stats(info)[0]
        assert (st.n_cpu > 0) if placement == "host" else (st.n_cpu == 0 and st.n_gpu > 0), st
    moe.close()


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["mixtral", "deepseek", "qwen2"])
@pytest.mark.parametrize("T,placement", [(1, "gpu"), (1, "host"), (64, "gpu")])
def test_b200_layer_matches_transformers_at_released_shapes(family, T, placement):
    """The released model shapes (Mixtral 4096 x 14336 top-2, DeepSeek-V2-Lite
    2048 x 1408 top-6 + 2 shared, Qwen2-57B 3584 x 2560 top-8 + 8-chunk gated
    shared expert), the transformers block evaluated on the GPU in fp32 (no
    TF32), against the B200 layer at bf16 tolerance."""
    from paper_2504_05897_b200.moe import layer_stats
    torch.backends.cuda.matmul.allow_tf32 = False
    Hf, If, n, k = FULL[family]
    blk, n, k, s_int = _block(family, 5 + T, FULL[family], device="cuda")
    moe, router, sgate = _hybrid(family, blk, n, k, s_int, T, 1e-3 if placement == "host" else 1e3, Hf, If)
    x = torch.randn(T, Hf, device="cuda").to(torch.bfloat16)
    with torch.no_grad():
        want = blk(x.float().reshape(1, T, Hf)).reshape(T, Hf).cpu().numpy()
    lg = torch.from_numpy(_logits(x.float(), router, sgate)).cuda()
    del blk
    torch.cuda.empty_cache()
    y, info = moe.forward_pass(x, [lg])
    torch.cuda.synchronize()
    got = y.float().cpu().numpy()
    assert np.abs(got - want).max() / np.abs(want).max() <= 1e-2
    st = layer_stats(info)[0]
    assert (st.n_cpu > 0) if placement == "host" else (st.n_cpu == 0 and st.n_gpu > 0), st
    moe.close()
