"""Summarise ncu outputs into profiles/ (launch-list shares + key metrics of a --set full capture).

    python tools/ncu_summary.py launches gpurun_out/launches.csv
    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep [alg_flops_per_launch]
    python tools/ncu_summary.py traffic out.json rep1.ncu-rep [rep2.ncu-rep ...]
        per-kernel DRAM bytes (read + write) per launch from --set full captures,
        keyed by the names bench.py profiles under (read by bench.py for
        roofline.traffic)
"""
import json
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "sm__cycles_active.avg",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].strip()[:70]
        v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    s2 = {k: v for k, v in agg.items() if "s2dev" in k}
    tot = sum(v[1] for v in s2.values())
    print("| kernel | launches | avg ms (cold, serialised) | share of S2 step |")
    print("|---|---|---|---|")
    for k, (n, t) in s2.items():
        print(f"| `{k}` | {n} | {t / n:.3f} | {t / tot:.1%} |")


def report(path, alg=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"### `{name[:90]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        got = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                got[k] = (vals[i], units[i])
                print(f"| {k} | {vals[i]} | {units[i]} |")
        if "dram__bytes_read.sum" in got:
            def to_bytes(v, u):
                f = float(v.replace(",", ""))
                return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            tr = to_bytes(*got["dram__bytes_read.sum"]) + to_bytes(*got["dram__bytes_write.sum"])
            print(f"| traffic (read+write) | {tr:.4e} | byte |")
        if alg and "gpu__time_duration.sum" in got:
            v, u = got["gpu__time_duration.sum"]
            t = float(v.replace(",", "")) * {"ms": 1e-3, "msecond": 1e-3, "us": 1e-6,
                                              "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9}.get(u, 1e-3)
            print(f"| algorithmic TFLOP/s under ncu (cold) | {float(alg) / t / 1e12:.1f} | TFLOP/s |")
        print()


BENCH_NAMES = {"s2_fwd_sm100_kernel": "fwd_sm100", "s2_bwd_dkv_kernel": "bwd_dkv_sm100",
               "s2_bwd_dq_kernel": "bwd_dq_sm100", "s2_bwd_prep_kernel": "bwd_prep",
               "s2_decode_split_kernel": "decode_split", "s2_decode_combine_kernel": "decode_combine"}


def traffic(out_path, reps):
    res = {}
    for path in reps:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for vals in rows[2:]:
            full = vals[hdr.index("Kernel Name")]
            key = next((v for k, v in BENCH_NAMES.items() if k in full), None)
            if key is None:
                continue

            def val(m):
                i = hdr.index(m)
                f = float(vals[i].replace(",", ""))
                return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                            "ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6,
                            "ns": 1e-9, "nsecond": 1e-9}.get(units[i], 1)
            res[key] = {"dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                        "duration_s_under_ncu": val("gpu__time_duration.sum"), "source": path.split("/")[-1]}
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
