"""Measure tcgen05.mma throughput per shape on one SM (probe library)."""
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(HERE, "tests", "cuda", "libumma_probe.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                       "-Xcompiler", "-fPIC", "-shared", "-o", so, os.path.join(HERE, "tests", "cuda", "umma_probe.cu")])
L = ctypes.CDLL(so)
out = (ctypes.c_longlong * 2)()
for kind, name in ((0, "SS"), (1, "TS")):
    for N in (64, 128, 256):
        iters = 4096
        assert L.probe_rate(kind, N, iters, out) == 0
        cyc = out[1] / iters
        ideal = 128 * N / 256
        print(f"{name} M=128 N={N:3d} K=16: {cyc:6.1f} cyc/MMA (issue {out[0]/iters:5.1f}), ideal {ideal:5.1f} -> {ideal/cyc:.0%}")
for variant, name in ((0, "S,dP + dV,dK"), (1, "S,dP only"), (2, "dV,dK only"), (3, "all + concurrent TMEM loads"), (4, "all + concurrent TMEM ld+st"), (5, "all + concurrent TMA 32KB loads"), (6, "all + 7 ALU-busy warps (issuer = lowest wid)"), (7, "commit after S,dP"), (8, "commit after S,dP and after dV,dK"), (9, "fence::after_thread_sync between groups"), (10, "commit+wait+fence between groups (drain)"), (11, "Q/dO tiles rotate between 2 stages")):
    assert L.probe_dkv_seq(512, variant, out) == 0
    print(f"dkv step sequence [{name}]: {out[0]/512:.0f} cyc/step")
modes = ["SS64 1acc", "SS64 2acc interleaved", "SS64 2acc grouped", "SS128 interleaved", "SS128 grouped",
         "TS128 2acc interleaved", "SS256 interleaved", "SS64 interleaved acc0-first", "SS64 grouped acc0-first"]
for m, name in enumerate(modes):
    if m == 6:
        continue
    assert L.probe_mix(m, 256, out) == 0
    n = 256 * 16
    N = 128 if m in (3, 4, 5) else (256 if m == 6 else 64)
    print(f"mix [{name}]: {out[1]/n:6.1f} cyc/MMA (ideal {N/2:.0f}), issue {out[0]/n:6.1f}")
for v, name in ((1, "S,dP"), (2, "dV,dK"), (3, "all"), (7, "all + TMEM ld/st"), (11, "all + TMA"), (15, "all + TMEM + TMA")):
    assert L.probe_dkv2(512, v, out) == 0
    print(f"dkv2 [{name}]: {out[0]/512:.0f} cyc/step (ideal S,dP 512 + dV,dK 512)")
for nw in (1, 4, 8, 16):
    it = 256
    assert L.probe_tmem_ld(nw, it, out) == 0
    by = nw * it * 4 * 32 * 32 * 4
    print(f"tmem ld: {nw:2d} warps: {out[0]/it:7.1f} cyc per 4 x x32 per warp; {by/out[0]:6.1f} B/cycle/SM")
