"""Hybrid layer stacks: the per-layer layout of a
LayerSchedule equals the reference's build_layer_masks (pattern.cpp:168-181)
— dense layer ids get the dense-causal mask, the others the sparse pattern —
and the stack hands each layer the plan with that layout.  CPU only (layout);
the GPU half is in test_gpu_fwd.py::test_hybrid_layer_stack."""
import numpy as np
import pytest

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200.pattern import LayerSchedule, make_single_stride_config


def test_layer_stack_maps_layers_to_the_reference_masks():
    pat = make_single_stride_config(2048, 64, 4, 2, 4)
    sched = LayerSchedule(6, {0, 3}, pat)
    stack = s2.LayerStack(sched)
    masks = s2.build_layer_masks(sched)
    B = pat.num_blocks()
    for layer in range(6):
        plan = stack.plan(layer)
        assert stack.is_dense(layer) == (layer in {0, 3})
        for h in range(4):
            assert plan.head_nnz(h) == masks[layer][h].popcount()
        if layer in {0, 3}:
            assert plan.stats()["nnz_total"] == 4 * B * (B + 1) // 2
    assert stack.plan(1) is stack.plan(2) and stack.plan(0) is stack.plan(3)


def test_layer_stack_rejects_bad_schedules():
    pat = make_single_stride_config(512, 64, 4, 1, 4)
    with pytest.raises(s2.S2InvalidArgument, match="outside"):
        s2.LayerStack(LayerSchedule(2, {2}, pat))
    with pytest.raises(s2.S2InvalidArgument, match="num_layers"):
        s2.LayerStack(LayerSchedule(0, set(), pat))
    stack = s2.LayerStack(LayerSchedule(2, set(), pat))
    with pytest.raises(s2.S2InvalidArgument):
        stack.plan(5)


def test_cfg3_hybrid_flops_match_the_schedule():
    """cfg3: 24 layers, dense {0, 1} — the speedup-vs-dense shape of the paper."""
    pat = s2.make_s2_config(32768, 32, local_blocks=4, vert_stride=16)
    stack = s2.LayerStack(LayerSchedule(24, {0, 1}, pat))
    a_s, d_s = stack.plan(5).fwd_flops(1, 128)
    a_d, d_d = stack.plan(0).fwd_flops(1, 128)
    assert a_d == d_d == d_s
    total = 2 * a_d + 22 * a_s
    assert 6.0 < 24 * d_s / total < 7.0  # 753 ms all-dense vs 116 ms ideal mix
