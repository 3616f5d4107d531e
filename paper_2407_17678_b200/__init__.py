"""B200-native S2-Attention (arXiv 2407.17678): layout builder, sm_100a
forward/backward/decode kernels and a head-parallel partitioner behind the C
ABI of include/s2attn.h (libs2attn.so, built in-tree)."""
from ._abi import S2ConfigError, S2Error, S2InvalidArgument, S2Unsupported, lib  # noqa: F401
from .pattern import (  # noqa: F401
    CsrMask, HeadBlockMask, LayerSchedule, PatternConfig, StrideSegment, build_all_csr,
    build_all_masks, build_csc, build_csr, build_head_mask, build_layer_masks,
    dense_causal_mask, evict_after, from_csr, kv_efficient, make_dense_config,
    make_multi_stride_config, make_s2_config, make_single_stride_config,
    make_sliding_window_config, nnz, same_bits, to_csr)
from .attention import (  # noqa: F401
    AttentionTensors, Plan, dsplit_attention, s2_attention, s2_attn_bwd, s2_attn_fwd, s2_attn_fwd_bwd_host, s2_attn_fwd_peers,
    streaming_sharded_attention)
from .serialize import (  # noqa: F401
    CliConfigFile, config_hash, csr_from_json, layer_schedule_from_json, load_config_file,
    pattern_config_from_json, to_json)
from .analysis import (  # noqa: F401
    CacheSchedule, FlopsReport, HeadCacheSchedule, analytic_flops_reduction,
    equivalent_context_length, exact_flops, flops_per_block_pair, kv_reduction,
    simulate_decode_cache, speedup_upper_bound)
from .layers import LayerStack  # noqa: F401
