#!/usr/bin/env python
"""bench.py — S2-Attention on B200 (BASELINE.json metric:
"S2 attn fwd+bwd ms & active-block TFLOPS @32K; decode tok/s; vs CPU ref").

A step = one S2 attention layer forward + backward over one batch of
synthetic bf16 inputs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl s2|reference]
                    [--workload cfg3|cfg5]

--workload cfg3 (default): BASELINE.json configs[2] (S=32K, H=32, D=128, block
    64, local_blocks 4, vert_stride 16, heterogeneous head offsets), one layer per
    GPU.  Under torchrun a global batch of N sequences is sharded one sequence
    per rank (weak scaling, data parallel): every rank owns complete outputs, so
    there is no data-path collective (--exchange allgather / fused add the
    head-parallel output exchange for comparison).
--workload cfg5: BASELINE.json configs[4] (S=128K, H=32, D=128, B=1), its 32
    heads LPT-split over the ranks by active blocks (strong scaling), all-gather
    of O overlapping the backward.

value          whole-job active-block TFLOP/s of fwd+bwd (FLOPs_fwd = sum nnz *
               4*D*64^2, analysis.cpp:29-31; FLOPs_bwd = 2.5 x FLOPs_fwd),
               device time (CUDA events), max over ranks, inputs resident in HBM.
e2e            the same through the public API with host buffers: H2D of q,k,v,dO
               from pinned memory and D2H of out,lse,dq,dk,dv inside the timed region.
roofline       dominant kernel of the step (CUDA events around every launch, via
               s2_profile_*, in a separate pass), algorithmic FLOPs / its average
               launch time.
clocks         SM clock / throttle reasons sampled every ~1 ms by a separate process
               (NVML) and kept when they fall inside the timed region.
cpu_baseline   the reference's streaming_sharded_attention (oracle/_ref, built from
               /root/reference) for the forward + the oracle's C restatement of the
               backward (the reference has none), on a bounded sample of cfg3 heads.
configs        (N=1) the other BASELINE configs, each with its roofline and CPU
               baseline: cfg1 fp32 forward (the reference's own bench config, run in
               full on both sides), cfg2 (B=4, 8K) and cfg5 (128K) fwd+bwd.
decode         cfg4 decode step (B=64, 128K context, 32q/8kv) over the compacted cache.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SEQ, H, D, BLOCK, LOCAL, VSTRIDE = 32768, 32, 128, 64, 4, 16
N_CFG5 = 131072
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
COMM_SMS = 16  # SMs the backward leaves to NCCL when N > 1
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (tools/ncu_summary.py traffic), or None."""
    try:
        with open(TRAFFIC_PATH) as f:
            return json.load(f)[kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def use_all_host_threads():
    """The CPU legs run on every host core. torchrun exports OMP_NUM_THREADS=1, so the
    variable is overridden (not defaulted), and the thread count is set directly on
    the libgomp that oracle/ links, in case it has already read its environment.
    Returns the thread count in effect, which is what `cores` reports."""
    n = host_cores()
    os.environ["OMP_NUM_THREADS"] = str(n)
    try:
        gomp = ctypes.CDLL("libgomp.so.1")
        gomp.omp_set_num_threads(ctypes.c_int(n))
        return int(gomp.omp_get_max_threads())
    except OSError:
        return n


# ---------------------------------------------------------------- CPU side
# Test / baseline infrastructure only: oracle/ (the reference compiled from its
# sources, and the C restatement of the backward).  Nothing here imports the
# product package, so the reference arm maps none of its libraries.
def _oracle():
    p = os.path.join(ROOT, "oracle")
    if p not in sys.path:
        sys.path.insert(0, p)
    import oracle

    return oracle


def cpu_sample(seq_len=N_SEQ, num_heads=H, d=D, vstride=VSTRIDE, heads=(0,), band=1.0, seed=7, bwd=True):
    """Time the reference CPU path on a bounded sample of a single-stride config:
    the forward through the reference library (or the port if it is absent), the
    backward through the port (the reference has none).  band < 1 keeps only a
    centred band of that fraction of the query blocks (the other rows' CSR lists
    are emptied; rows in the middle of the sequence have the average row length).
    The layout is the reference's own to_csr(build_all_masks).
    Returns (tflops, seconds, kind, sample_desc, flops)."""
    threads = use_all_host_threads()
    oracle = _oracle()
    c = oracle.single_stride(seq_len, BLOCK, num_heads, LOCAL, vstride)
    rp_all, ci_all, _ = oracle.csr_all_c(c)
    B = (seq_len + BLOCK - 1) // BLOCK
    nnz = [int(rp_all[h * (B + 1) + B]) for h in range(num_heads)]
    offs = np.concatenate([[0], np.cumsum(nnz)])
    ref = oracle.ref()
    kind = "reference" if ref is not None else "port"
    rng = np.random.default_rng(seed)
    tot_s = 0.0
    flops = 0.0
    for h in heads:
        rp = np.ascontiguousarray(rp_all[h * (B + 1):(h + 1) * (B + 1)], np.int32)
        ci = np.ascontiguousarray(ci_all[offs[h]:offs[h + 1]], np.int32)
        if band < 1.0:
            nb = max(1, int(round(B * band)))
            r0 = (B - nb) // 2
            lens = np.diff(rp)
            keep = np.zeros(B, bool)
            keep[r0:r0 + nb] = True
            ci = np.ascontiguousarray(ci[np.repeat(keep, lens)], np.int32)
            rp = np.concatenate([[0], np.cumsum(np.where(keep, lens, 0))]).astype(np.int32)
        n = seq_len * d
        q, k, v, do = (rng.uniform(-1, 1, n).astype(np.float32) for _ in range(4))
        out = np.zeros(n, np.float32)
        lse = np.zeros(seq_len, np.float64)
        t0 = time.perf_counter()
        if ref is not None:
            rc = ref.ref_streaming(1, seq_len, d, BLOCK, 0.0, oracle.fp(q), oracle.fp(k), oracle.fp(v),
                                   B, oracle.ip(rp), oracle.ip(ci), 0, oracle.fp(out), oracle.dp(lse))
            assert rc == 0
        else:
            oracle.attn_fwd(q, k, v, rp, ci, 1, 1, 1, seq_len, d, BLOCK)
        if bwd:
            oracle.attn_bwd_par(q, k, v, do, rp, ci, 1, 1, 1, seq_len, d, BLOCK)
        tot_s += time.perf_counter() - t0
        flops += (3.5 if bwd else 1.0) * int(ci.size) * 4.0 * d * BLOCK * BLOCK
    desc = (f"S={seq_len} H={num_heads} D={d} v={vstride}: heads {list(heads)} of {num_heads}"
            + (f", centred band of {band:g} of the query blocks" if band < 1 else "")
            + f" (fwd: {'reference streaming_sharded_attention' if kind == 'reference' else 'oracle port'}"
            + ("; bwd: oracle C restatement parallel over rows and key blocks, the reference has no backward"
               if bwd else "") + f"), fp32/fp64, {threads} threads")
    return flops / tot_s / 1e12, tot_s, kind, desc, flops


def reference_cfg1_full():
    """The reference's own benchmark config (bench_attention.cpp:30-34: cfg1, fp32
    H=8 N=2048 D=64, local 4, v=8, seed 7) run in FULL by the reference library:
    the forward all heads at once (its OpenMP head loop), ms."""
    threads = use_all_host_threads()
    oracle = _oracle()
    ref = oracle.ref()
    c = oracle.single_stride(2048, BLOCK, 8, 4, 8)
    rp, ci, _ = oracle.csr_all_c(c)
    q, k, v = oracle.random_tensors(8, 2048, 64, 7)
    out = np.zeros(q.size, np.float32)
    lse = np.zeros(8 * 2048, np.float64)
    B = 32
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        if ref is not None:
            assert ref.ref_streaming(8, 2048, 64, BLOCK, 0.0, oracle.fp(q), oracle.fp(k), oracle.fp(v), B,
                                     oracle.ip(rp), oracle.ip(ci), 0, oracle.fp(out), oracle.dp(lse)) == 0
        else:
            oracle.attn_fwd(q, k, v, rp, ci, 1, 8, 8, 2048, 64, BLOCK)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    flops = int(ci.size) * 4.0 * 64 * BLOCK * BLOCK
    return {"ms": best * 1e3, "tflops": flops / best / 1e12, "cores": threads,
            "kind": "reference" if ref is not None else "port",
            "sample": "cfg1 in full: fp32 forward of all 8 heads (bench_attention.cpp's config), best of 3"}


def reference_workload_desc(band):
    return {"workload": f"cfg3 SAMPLE per step: one head of S=32768 H=32 D=128 (block 64, local_blocks 4, "
                        f"vert_stride 16, heterogeneous offsets), centred band of {band:g} of its query blocks; "
                        "fwd = the reference's streaming_sharded_attention, bwd = the oracle's C restatement "
                        "(the reference has none)",
            "seq_len": N_SEQ, "heads_sampled_per_step": 1, "head_dim": D, "parallelism": "OpenMP, host cores"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    use_all_host_threads()
    band = 1.0 / 2
    # bounded steps: a 1/2 band of one head per step (~1-2 s on 16 cores), warm-up 1/16
    for _ in range(args.warmup):
        cpu_sample(heads=(0,), band=1.0 / 16)
    vals, secs = [], []
    kind = desc = None
    for i in range(args.steps):
        v, s, kind, desc, _ = cpu_sample(heads=(i % H,), band=band)
        vals.append(v)
        secs.append(s)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": "S2 attn fwd+bwd active-block TFLOP/s @32K",
        "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": reference_workload_desc(band),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": use_all_host_threads(), "kind": kind,
                         "sample": desc + "; one head band per step"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_desc(n, exchange="none"):
    if exchange == "none":
        par = f"data-parallel x{n}: one sequence per GPU, no collective on the data path"
    else:
        how = ("forward stores O into every rank's output (fused exchange)" if exchange == "fused" and n > 1
               else "all-gather of O")
        par = f"head-parallel x{n} (LPT by active blocks), {how}"
    return {"workload": "cfg3: one S2 attention layer fwd+bwd, S=32768, H=32, D=128, block 64, "
                        "local_blocks 4, vert_stride 16, heterogeneous head offsets",
            "batch_per_gpu": 1, "global_batch": n, "seq_len": N_SEQ, "heads": H, "head_dim": D,
            "parallelism": par,
            "l2": "inputs 256 MiB per tensor > 126 MB L2; no flush needed"}


# ------------------------------------------------------------- clock sampler
_SAMPLER = r"""
import signal, sys, time
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
end = time.monotonic() + float(sys.argv[2])
stop = []
signal.signal(signal.SIGTERM, lambda *a: stop.append(1))
print("ready", flush=True)
buf = []
while time.monotonic() < end and not stop:
    t = time.monotonic()
    try:
        buf.append("%.6f %d %d" % (t, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                   nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
    except Exception:
        pass
    time.sleep(float(sys.argv[3]))
    if len(buf) >= 200000:
        break
sys.stdout.write("\n".join(buf) + "\n")
sys.stdout.flush()
"""


class ClockSampler:
    """SM clock and throttle reasons from a separate process polling NVML every
    ~1 ms (a thread in this process starves behind the launch loop's GIL), kept
    when they fall inside the timed region [mark_start(), mark_end()]
    (time.monotonic is system-wide)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, dev_index, max_seconds=600.0):
        self.max_mhz, self.samples, self.reasons = None, [], set()
        self.t0 = self.t1 = None
        self.proc = None
        try:
            import pynvml

            pynvml.nvmlInit()
            idx = self._nvml_index(pynvml, dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(idx),
                                                            pynvml.NVML_CLOCK_SM)
            period = float(os.environ.get("S2_CLOCK_PERIOD_MS", "0.5")) * 1e-3
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(idx), str(max_seconds), str(period)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            if self.proc.stdout.readline().strip() != "ready":
                self.proc = None
        except Exception:
            self.proc = None

    @staticmethod
    def _nvml_index(nv, dev_index):
        import torch

        try:
            uuid = str(torch.cuda.get_device_properties(dev_index).uuid).replace("GPU-", "")
            for i in range(nv.nvmlDeviceGetCount()):
                u = nv.nvmlDeviceGetUUID(nv.nvmlDeviceGetHandleByIndex(i))
                u = u.decode() if isinstance(u, bytes) else u
                if uuid and uuid in u:
                    return i
        except Exception:
            pass
        return dev_index

    def mark_start(self):
        self.t0 = time.monotonic()

    def mark_end(self):
        self.t1 = time.monotonic()

    def finish(self):
        if self.proc is None:
            return
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=30)
        except Exception:
            self.proc.kill()
            out = ""
        # SIGTERM ends the sampler's loop; it then prints its buffer
        for ln in (out or "").splitlines():
            p = ln.split()
            if len(p) != 3:
                continue
            t, mhz, r = float(p[0]), int(p[1]), int(p[2])
            if self.t0 is not None and self.t1 is not None and self.t0 <= t <= self.t1:
                self.samples.append(mhz)
                for k, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(k)

    def summary(self):
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples),
                "sm_mhz_range": [min(self.samples), max(self.samples)] if self.samples else None,
                "how": "NVML from a separate process, ~1 ms period, samples inside the timed region"}


# --------------------------------------------------------------------- GPU side
def _kernel_profile(lib, fn, steps, barrier):
    """Per-kernel averages over `steps` calls of fn with CUDA events around every
    launch (a separate pass: events between launches serialise the programmatic
    dependent launches the timed loop relies on)."""
    lib.s2_profile_enable(1)
    for _ in range(steps):
        fn()
    barrier()
    names = ctypes.create_string_buffer(32 * 16)
    tot = (ctypes.c_double * 16)()
    cnt = (ctypes.c_int * 16)()
    nk = ctypes.c_int()
    lib.s2_profile_collect(16, names, tot, cnt, ctypes.byref(nk))
    lib.s2_profile_enable(0)
    kernels = {}
    for i in range(nk.value):
        nm = names.raw[32 * i: 32 * i + 32].split(b"\0")[0].decode()
        kernels[nm] = {"avg_ms": tot[i] / cnt[i], "launches": cnt[i]}
    return kernels


def _roofline(kernels, fwd_flops, pk, pk_kind, with_traffic=True):
    """Roofline of the dominant kernel; algorithmic FLOPs per launch:
    fwd_sm100: F; bwd_dkv: S-recompute + dP + dV + dK = 2F; bwd_dq: dQ = 0.5F.
    traffic: the committed ncu capture is of the cfg3 workload only, so other
    workloads report null (with_traffic=False)."""
    alg = {"fwd_sm100": fwd_flops, "bwd_dkv_sm100": 2.0 * fwd_flops, "bwd_dq_sm100": 0.5 * fwd_flops,
           "bwd_prep": 0.0}
    dom = max(kernels, key=lambda k_: kernels[k_]["avg_ms"]) if kernels else None
    if not dom:
        return None
    ach = alg.get(dom, 0.0) / (kernels[dom]["avg_ms"] * 1e-3) / 1e12
    return {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops"],
            "unit": "TFLOP/s", "frac": ach / pk["bf16_tflops"],
            "traffic": ncu_traffic(dom) if with_traffic else None,
            "traffic_source": ("profiles/ncu_traffic.json (dram__bytes_read+write per launch, ncu --set full, cfg3)"
                               if with_traffic else "no ncu capture of this workload"),
            "peak_source": f"{pk_kind} bf16_tflops (burst)",
            "frac_of_sustained": ach / pk.get("bf16_tflops_sustained", pk["bf16_tflops"]),
            "alg_flops_per_launch": alg.get(dom, 0.0)}


def _setup_dist(collective: bool = True):
    import torch
    import torch.distributed as dist

    from paper_2407_17678_b200 import _abi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test-only switches (tests/test_gpu_multirank.py): S2_BENCH_SHARE_GPU=1 puts
    # every rank on cuda:0 and S2_BENCH_BACKEND=gloo replaces NCCL, so the
    # multi-rank path runs on a one-GPU box.  Never a performance configuration.
    if os.environ.get("S2_BENCH_SHARE_GPU") == "1":
        local = 0
    backend = os.environ.get("S2_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            # NCCL's all-gather CTAs share the GPU with the backward: cap them and keep
            # their SMs out of the backward kernels' grids (s2_set_sm_reserve; the
            # forward keeps every SM).  NCCL_DEBUG=INFO keeps its init log (rank count,
            # NVLS) visible on stderr.
            os.environ.setdefault("NCCL_MAX_CTAS", str(COMM_SMS))
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
            if collective:  # only a step with an exchange leaves NCCL its SMs
                _abi.check(_abi.lib().s2_set_sm_reserve(int(os.environ["NCCL_MAX_CTAS"])))
        else:
            dist.init_process_group(backend)
    return world, rank, local, dev


def run_s2(args):
    import torch
    import torch.distributed as dist

    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200 import _abi
    from paper_2407_17678_b200.dist import HeadParallelPlan

    world, rank, local, dev = _setup_dist(collective=args.exchange != "none")
    cfg5 = args.workload == "cfg5"
    n_seq = N_CFG5 if cfg5 else N_SEQ
    cfg = s2.make_s2_config(n_seq, H, block_size=BLOCK, local_blocks=LOCAL, vert_stride=VSTRIDE)
    plan = s2.Plan.from_config(cfg)
    # cfg3: global batch = world (weak scaling, one layer per GPU);
    # cfg5: one 128K sequence, its 32 heads split over the ranks (strong scaling)
    gbatch = 1 if cfg5 else world
    # cfg3 without an exchange: one whole sequence per rank (data parallel)
    hp = HeadParallelPlan(plan, gbatch, world, mode="batch" if args.exchange == "none" else "lpt")
    units = hp.units[rank]
    U = len(units)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    mk = lambda: torch.rand((U, 1, n_seq, D), device=dev, generator=g, dtype=torch.float32)  # noqa
    q, do = (mk().mul_(2).sub_(1).to(torch.bfloat16) for _ in range(2))
    k, v = (mk().mul_(2).sub_(1).to(torch.bfloat16).reshape(U, n_seq, D) for _ in range(2))
    out = torch.empty_like(q)
    lse = torch.empty((U, 1, n_seq), device=dev, dtype=torch.float32)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    act1, dense1 = plan.fwd_flops(1, D)
    w = plan.unit_weights(gbatch)
    per_pair = 4.0 * D * BLOCK * BLOCK
    my_fwd_flops = float(sum(w[u] for u in units)) * per_pair
    tot_fwd_flops = float(w.sum()) * per_pair
    dense_fwd_total = dense1 * gbatch

    fused = world > 1 and args.exchange == "fused"
    if fused:
        # the forward stores every O tile straight into each rank's full output
        # (peer memory); one tiny collective per step orders the ranks' kernels
        from paper_2407_17678_b200.dist import PeerOutputs

        peers = PeerOutputs(hp, n_seq, D, torch.bfloat16, dev, rank)
        unit_global = torch.as_tensor(np.asarray(units, dtype=np.int32), device=dev)
        fence = torch.zeros(1, device=dev)

    def step():
        if fused:
            s2.s2_attn_fwd_peers(plan, q, k, v, unit_ids=units, peer_out=peers.peer_out, peer_lse=peers.peer_lse,
                                 unit_global=unit_global, total_units=peers.total_units, out=out, lse=lse)
            # the backward needs only this rank's units; the fence after it makes
            # every rank's forward (and so every peer write) complete
            s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv, unit_ids=units)
            dist.all_reduce(fence)
            return
        s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse, unit_ids=units)
        exchange = world > 1 and args.exchange != "none"
        finish = hp.all_gather_async(out.reshape(U, 1, n_seq, D)) if exchange else None
        # the backward needs only this rank's units: it overlaps the all-gather
        s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv, unit_ids=units)
        if finish is not None:
            finish()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clk = ClockSampler(local)
    for _ in range(args.warmup):
        step()
    barrier()
    lib = _abi.lib()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    clk.mark_start()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    clk.mark_end()
    clk.finish()
    ms = e0.elapsed_time(e1) / args.steps
    kernels = _kernel_profile(lib, step, args.steps, barrier)
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = 3.5 * tot_fwd_flops / (ms_max * 1e-3) / 1e12
    fwd_ms = kernels.get("fwd_sm100", {}).get("avg_ms", float("nan"))
    bwd_ms = sum(kernels.get(k_, {}).get("avg_ms", 0.0) for k_ in ("bwd_prep", "bwd_dkv_sm100", "bwd_dq_sm100"))
    pk, pk_kind = peaks()
    roof = _roofline(kernels, my_fwd_flops, pk, pk_kind, with_traffic=args.workload == "cfg3")

    if cfg5:
        cdesc = {"workload": "cfg5: one S2 attention layer fwd+bwd, S=131072, H=32, D=128, B=1, block 64, "
                             "local_blocks 4, vert_stride 16, heterogeneous head offsets",
                 "global_batch": 1, "seq_len": n_seq, "heads": H, "head_dim": D,
                 "parallelism": f"head-parallel x{world}: the 32 heads LPT-split by active blocks, "
                                "all-gather of O overlapping the backward",
                 "l2": "inputs 1 GiB per tensor > 126 MB L2; no flush needed"}
    else:
        cdesc = config_desc(world, args.exchange)
    line = {
        "metric": f"S2 attn fwd+bwd active-block TFLOP/s @{'128K' if cfg5 else '32K'}", "value": value,
        "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong" if cfg5 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (U[-1,1] bf16)", "config": cdesc,
        "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
        "dense_equiv_tflops": 3.5 * dense_fwd_total / (ms_max * 1e-3) / 1e12,
        "dense_causal_fwd_bwd_flops_per_gpu": 3.5 * dense1 * gbatch / world,
        "active_fwd_bwd_flops_per_gpu": 3.5 * my_fwd_flops,
        "kernels": kernels, "roofline": roof,
        "gpu_launches": int(sum(v_["launches"] for v_ in kernels.values())),
        "clocks": clk.summary(),
    }
    if world > 1 or cfg5:
        # the exchange budget: every rank receives the other ranks' O (bf16) once per step
        # (none in the data-parallel cfg3 mode)
        o_bytes = gbatch * H * n_seq * D * 2 if args.exchange != "none" else 0
        line["exchange"] = {"mode": args.exchange, "all_gather_bytes_total": o_bytes,
                            "received_bytes_per_gpu": o_bytes * (world - 1) // max(1, world),
                            "padded_send_bytes_per_gpu": hp.max_units * n_seq * D * 2 if o_bytes else 0,
                            "overlap_window_ms": bwd_ms,
                            "rank_active_blocks": [int(x) for x in hp.load],
                            "imbalance_max_over_ideal": hp.imbalance(),
                            "nccl_max_ctas": int(os.environ.get("NCCL_MAX_CTAS", "0")) if world > 1 else 0,
                            "sm_reserve_backward": (int(os.environ.get("NCCL_MAX_CTAS", "0"))
                                                    if world > 1 and args.exchange != "none" else 0)}

    # ---- end to end through the public API with host buffers
    if not args.no_e2e and not cfg5:
        line["e2e"] = bench_e2e(s2, plan, args, world, U, q, k, v, do, out, lse, dq, dk, dv, step, barrier,
                                tot_fwd_flops, dev)

    # ---- hybrid 24-layer mix of cfg3 (dense layers {0, 1}, configs/l1v15_dense01.json
    #      shape): one dense-causal layer through the same kernels (LayerStack),
    #      the mix = 2 dense + 22 S2 layers vs 24 dense layers (PAPER speedup shape)
    if not args.no_hybrid and world == 1 and not cfg5:
        try:
            line["hybrid"] = bench_hybrid(s2, cfg, q, k, v, do, ms_max, dev)
        except Exception as ex:  # reported, never fatal to the main number
            line["hybrid"] = {"error": str(ex)}

    # ---- decode at cfg4 (B=64, 128K context, GQA 32q/8kv, v=8), per GPU
    if not args.no_decode and not cfg5:
        try:
            line["decode"] = bench_decode(args, dev, world)
        except Exception as ex:  # reported, never fatal to the main number
            line["decode"] = {"error": str(ex)}

    # ---- the other BASELINE configs (N=1): cfg1 fp32, cfg2, cfg5
    if not args.no_configs and world == 1 and not cfg5:
        del q, k, v, do, out, lse, dq, dk, dv
        torch.cuda.empty_cache()
        line["configs"] = bench_configs(s2, args, dev, lib, pk, pk_kind, not args.no_cpu_baseline)

    # ---- CPU baseline (rank 0, N=1 only)
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            threads = use_all_host_threads()
            val, secs, kind, desc, fl = cpu_sample(seq_len=n_seq, heads=tuple(range(8)) if not cfg5 else (0,),
                                                   band=1.0 if not cfg5 else 0.25)
            line["cpu_baseline"] = {"value": val, "unit": "TFLOP/s", "cores": threads,
                                    "kind": kind, "sample": desc, "seconds": secs}
        except Exception as ex:  # reported, never fatal to the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(ex)}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def bench_e2e(s2, plan, args, world, U, q, k, v, do, out, lse, dq, dk, dv, step, barrier, tot_fwd_flops, dev):
    import torch
    import torch.distributed as dist

    pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)  # noqa
    hq, hk, hv, hdo = pin(q), pin(k), pin(v), pin(do)
    ho, hl, hdq, hdk, hdv = (torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (out, lse, dq, dk, dv))
    e2e_steps = max(1, min(args.steps, 5))
    chunks = int(os.environ.get("S2_E2E_CHUNKS", "32"))
    e2e_api = (f"s2_attn_fwd_bwd_host (C ABI, host buffers, H2D/kernels/D2H pipelined over "
               f"{chunks} unit chunks)")
    if world == 1:
        # the host-resident data path of the public API: one call per step
        hq4, hk4, hv4, hdo4 = (t.reshape(1, U, N_SEQ, D) for t in (hq, hk, hv, hdo))
        ho4, hdq4 = ho.reshape(1, U, N_SEQ, D), hdq.reshape(1, U, N_SEQ, D)
        hl4 = hl.reshape(1, U, N_SEQ)
        hdk4, hdv4 = hdk.reshape(1, U, N_SEQ, D), hdv.reshape(1, U, N_SEQ, D)
        ws_holder = [None]

        def e2e_step():
            ws_holder[0] = s2.s2_attn_fwd_bwd_host(plan, hq4, hk4, hv4, hdo4, ho4, hl4, hdq4, hdk4, hdv4,
                                                   num_chunks=chunks, workspace=ws_holder[0])
    else:
        e2e_api = "torch copies from pinned host memory + s2_attn_fwd/bwd on this rank's units"

        def e2e_step():
            q.copy_(hq, non_blocking=True)
            k.copy_(hk, non_blocking=True)
            v.copy_(hv, non_blocking=True)
            do.copy_(hdo, non_blocking=True)
            step()
            for dst, src in ((ho, out), (hl, lse), (hdq, dq), (hdk, dk), (hdv, dv)):
                dst.copy_(src, non_blocking=True)

    e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e2e_steps):
        e2e_step()
    e1.record()
    barrier()
    ems = torch.tensor([e0.elapsed_time(e1) / e2e_steps], device=dev)
    if world > 1:
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
    ems = float(ems.item())
    h2d = sum(t.numel() * t.element_size() for t in (q, k, v, do))
    d2h = sum(t.numel() * t.element_size() for t in (out, lse, dq, dk, dv))
    return {"value": 3.5 * tot_fwd_flops / (ems * 1e-3) / 1e12, "unit": "TFLOP/s",
            "ms_per_step": ems, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": e2e_api, "pcie": pcie_bound(ho, hdq, out, dq, h2d, d2h, ems)}


def pcie_bound(h_a, h_b, d_a, d_b, h2d, d2h, ems):
    """The e2e path's floor on this box: pinned copies in both directions at once
    (H2D into d_a while D2H out of d_b), measured here on scratch buffers of the
    step's own tensors."""
    import torch

    s1, s2_ = torch.cuda.Stream(), torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def both():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2_.wait_event(ev)
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)
        with torch.cuda.stream(s2_):
            h_b.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2_)

    both()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        both()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    nbytes = h_a.numel() * h_a.element_size() + h_b.numel() * h_b.element_size()
    gbs = nbytes / (ms * 1e-3) / 1e9
    floor = (h2d + d2h) / (gbs * 1e9) * 1e3
    return {"duplex_gbs": gbs, "floor_ms": floor, "frac_of_floor": floor / ems,
            "note": "pinned H2D and D2H at once (the bytes of a step move no faster than this)"}


def _time_steps(fn, steps, warmup):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def bench_configs(s2, args, dev, lib, pk, pk_kind, with_cpu):
    """The other BASELINE configs on one GPU, each timed like the main step
    (CUDA events, warm-up, inputs resident), with its roofline and CPU baseline."""
    import torch

    res = {}
    steps, warm = max(3, min(args.steps, 10)), max(3, min(args.warmup, 3))
    g = torch.Generator(device=dev).manual_seed(77)
    uni = lambda shape, dt=torch.bfloat16: (torch.rand(shape, device=dev, generator=g) * 2 - 1).to(dt)  # noqa

    # cfg1: the reference's own bench config, fp32 forward (reference precision, SIMT
    # kernel), run in full on both sides: GPU vs the reference library on the host cores
    try:
        cfg = s2.make_s2_config(2048, 8, block_size=BLOCK, local_blocks=4, vert_stride=8)
        plan = s2.Plan.from_config(cfg)
        q, k, v = (uni((1, 8, 2048, 64), torch.float32) for _ in range(3))
        out, lse = s2.s2_attn_fwd(plan, q, k, v)
        ms = _time_steps(lambda: s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse), 20, 3)
        act, _ = plan.fwd_flops(1, 64)
        pk_, _src = peaks()
        mhz = float(pk_.get("sm_max_mhz", 1965.0))
        fp32_peak = 148 * 128 * 2 * mhz * 1e6 / 1e12  # FFMA lanes x 2 flops x clock
        ach = act / (ms * 1e-3) / 1e12
        r = {"workload": "cfg1: fp32 forward B=1 H=8 S=2048 D=64, block 64, local 4, vert_stride 8",
             "dtype": "f32", "ms": ms, "tflops_active": ach,
             "kernel": "s2_fwd_tile_kernel (fp32 FFMA from shared-memory tiles, the 1e-4 parity path)",
             "roofline": {"bound": "fp32 FFMA (SIMT)", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
                          "frac": ach / fp32_peak, "traffic": None,
                          "peak_source": "derived: 148 SMs x 128 FFMA/clk x 2 x sm_max_mhz (not measured)",
                          "alg_flops_per_launch": act}}
        if with_cpu:
            cb = reference_cfg1_full()
            r["cpu_baseline"] = cb
            r["gpu_speedup_vs_reference"] = cb["ms"] / ms
        res["cfg1_fp32_fwd"] = r
        del q, k, v, out, lse
    except Exception as ex:
        res["cfg1_fp32_fwd"] = {"error": str(ex)}

    # cfg2 (B=4 H=32 8K) and cfg5 (B=1 H=32 128K), bf16 fwd+bwd
    for name, B_, N_ in (("cfg2_b4_8k", 4, 8192), ("cfg5_128k", 1, N_CFG5)):
        try:
            cfg = s2.make_s2_config(N_, H, block_size=BLOCK, local_blocks=LOCAL, vert_stride=VSTRIDE)
            plan = s2.Plan.from_config(cfg)
            q, k, v, do = (uni((B_, H, N_, D)) for _ in range(4))
            out, lse = s2.s2_attn_fwd(plan, q, k, v)
            dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)

            def st():
                s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
                s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv)

            ms = _time_steps(st, steps, warm)
            kern = _kernel_profile(lib, st, steps, torch.cuda.synchronize)
            act, dense = plan.fwd_flops(B_, D)
            r = {"workload": f"{name}: bf16 fwd+bwd B={B_} H=32 S={N_} D=128, block 64, local 4, vert_stride 16",
                 "dtype": "bf16", "ms_per_step": ms, "tflops_active": 3.5 * act / (ms * 1e-3) / 1e12,
                 "dense_equiv_tflops": 3.5 * dense / (ms * 1e-3) / 1e12, "kernels": kern,
                 "roofline": _roofline(kern, act, pk, pk_kind, with_traffic=False)}
            if with_cpu:
                v_, s_, kind, desc, _ = cpu_sample(seq_len=N_, heads=(0,), band=1.0 if N_ <= 8192 else 0.125)
                r["cpu_baseline"] = {"value": v_, "unit": "TFLOP/s", "cores": use_all_host_threads(), "kind": kind,
                                     "sample": desc, "seconds": s_}
            res[name] = r
            del q, k, v, do, out, lse, dq, dk, dv
            torch.cuda.empty_cache()
        except Exception as ex:
            res[name] = {"error": str(ex)}
    return res


def bench_decode(args, dev, world):
    """cfg4 decode step: 64 sequences x 1 token at position 131071 over the
    compacted cache; tok/s and achieved HBM GB/s (bytes = retained K/V + q/out)."""
    import torch

    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200 import _abi
    from paper_2407_17678_b200.decode import KVCache

    Bd, Hq, Hk, T = 64, 32, 8, 131072
    plan = s2.Plan.from_config(s2.make_s2_config(T, Hq, num_kv_heads=Hk, block_size=64,
                                                 local_blocks=4, vert_stride=8))
    cache = KVCache(plan, Bd, D)
    g = torch.Generator(device=dev).manual_seed(99)
    kv = torch.empty((Bd, Hk, T, D), device=dev, dtype=torch.bfloat16)
    kv.normal_(generator=g)
    cache.prefill(kv, kv)
    del kv
    torch.cuda.empty_cache()
    q = torch.randn((Bd, Hq, D), device=dev, dtype=torch.bfloat16, generator=g)
    out, lse = cache.decode(q)
    steps = max(args.steps, 20)
    lib = _abi.lib()
    # timed loop without per-launch events; the kernel split from a separate pass
    ms = _time_steps(lambda: cache.decode(q, out=out, lse=lse), steps, max(args.warmup, 3))
    kern = _kernel_profile(lib, lambda: cache.decode(q, out=out, lse=lse), steps, torch.cuda.synchronize)
    by = cache.decode_bytes()
    pool, dense = cache.bytes()
    pk, pk_kind = peaks()
    split_ms = kern.get("decode_split", {}).get("avg_ms", ms)
    ach = by / (split_ms * 1e-3) / 1e9
    # e2e: q from pinned host, out back to pinned host, every step
    hq = torch.empty(q.shape, dtype=q.dtype, pin_memory=True).copy_(q)
    ho = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)

    def e2e():
        q.copy_(hq, non_blocking=True)
        cache.decode(q, out=out, lse=lse)
        ho.copy_(out, non_blocking=True)

    ems = _time_steps(e2e, steps, 1)
    return {"metric": "decode tok/s (B=64, 128K ctx, 32q/8kv, v=8, compacted cache)",
            "value": world * Bd / (ms * 1e-3), "unit": "tok/s", "ms_per_step": ms,
            "kernels": kern, "bytes_per_step": by, "pool_bytes": pool, "dense_cache_bytes": dense,
            "roofline": {"kernel": "decode_split", "bound": "hbm", "achieved": ach,
                         "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ach / pk["hbm_gbs"],
                         "frac_of_8TBps": ach / 8000.0, "traffic": ncu_traffic("decode_split"),
                         "peak_source": f"{pk_kind} hbm_gbs",
                         "note": "decode_split time from the profiled pass; whole-step ms from the plain loop"},
            "e2e": {"value": world * Bd / (ems * 1e-3), "unit": "tok/s", "ms_per_step": ems,
                    "h2d_bytes_per_step": q.numel() * 2, "d2h_bytes_per_step": out.numel() * 2}}


def bench_hybrid(s2, cfg, q, k, v, do, s2_ms, dev, layers=24, dense_ids=(0, 1)):
    """Dense-causal fwd+bwd of one cfg3-shaped layer (the hybrid model's dense
    layers) through the LayerStack, CUDA events, then the 24-layer mix."""
    import torch

    from paper_2407_17678_b200.pattern import LayerSchedule

    stack = s2.LayerStack(LayerSchedule(layers, set(dense_ids), cfg))
    dl = dense_ids[0]
    U = q.shape[0]
    # full H=32 heads: the unit packing of the main bench holds one kv head per unit;
    # run the dense layer on the first 32 units' worth of rows re-viewed as heads.
    Hh = min(H, U)
    qd = q[:Hh].reshape(1, Hh, N_SEQ, D)
    kd, vd = (t[:Hh].reshape(1, Hh, N_SEQ, D) for t in (k, v))
    dod = do[:Hh].reshape(1, Hh, N_SEQ, D)
    plan = stack.plan(dl)
    o, l = torch.empty_like(qd), torch.empty((1, Hh, N_SEQ), device=dev, dtype=torch.float32)
    gq, gk, gv = torch.empty_like(qd), torch.empty_like(kd), torch.empty_like(vd)

    def dstep():
        s2.s2_attn_fwd(plan, qd, kd, vd, out=o, lse=l)
        s2.s2_attn_bwd(plan, qd, kd, vd, o, l, dod, dq=gq, dk=gk, dv=gv)

    dense_ms = _time_steps(dstep, 3, 2) * (H / Hh)
    act, dense_fl = plan.fwd_flops(1, D)
    nd = len(dense_ids)
    mix = nd * dense_ms + (layers - nd) * s2_ms
    return {"layers": layers, "dense_layer_ids": list(dense_ids), "dense_layer_ms": dense_ms,
            "s2_layer_ms": s2_ms, "hybrid_ms": mix, "all_dense_ms": layers * dense_ms,
            "speedup_vs_all_dense": layers * dense_ms / mix,
            "dense_layer_tflops": 3.5 * dense_fl * (Hh / H) / (dense_ms * (Hh / H) * 1e-3) / 1e12,
            "note": "fwd+bwd per layer, CUDA events; dense layers = make_dense_config through LayerStack"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="s2", choices=["s2", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg5"],
                    help="cfg3: S=32K layer per GPU (weak scaling, default); cfg5: one S=128K layer, heads "
                         "split over the GPUs (strong scaling)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-hybrid", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg1/cfg2/cfg5 lines (N=1)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "none", "allgather", "fused"],
                    help="N>1: none (cfg3 default: one sequence per rank, nothing to exchange), NCCL "
                         "all-gather of O overlapped with the backward (cfg5 default: one sequence's "
                         "heads over the ranks), or the forward storing O straight into every rank's "
                         "output (s2_attn_fwd_peers)")
    args = ap.parse_args()
    if args.exchange == "auto":
        args.exchange = "allgather" if args.workload == "cfg5" else "none"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_s2(args)


if __name__ == "__main__":
    main()
