"""bench.py's CPU legs (cpu_baseline and --impl reference) on the host cores: they
use every host thread even under torchrun (which exports OMP_NUM_THREADS=1), and
`cores` reports the thread count libgomp actually has."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpu_legs_override_torchrun_thread_default():
    code = (
        "import os, sys, ctypes; sys.path.insert(0, %r); import bench; "
        "n = bench.use_all_host_threads(); "
        "g = ctypes.CDLL('libgomp.so.1'); "
        "print(n, bench.host_cores(), os.environ['OMP_NUM_THREADS'], g.omp_get_max_threads())" % ROOT)
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    n, cores, var, gomp = (int(x) for x in r.stdout.split()[-4:])
    assert n == cores == var == gomp


def test_reference_arm_prints_one_line_with_its_thread_count():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    import json

    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    cores = len(os.sched_getaffinity(0))
    assert d["cpu_baseline"]["cores"] == cores and f"{cores} threads" in d["cpu_baseline"]["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_loads_nothing_from_the_product():
    """The reference arm runs the reference library and the oracle only: neither the
    product package nor its libraries are imported or mapped."""
    code = (
        "import sys, argparse; sys.path.insert(0, %r); import bench; "
        "bench.run_reference(argparse.Namespace(gpus=1, steps=1, warmup=0)); "
        "maps = open('/proc/self/maps').read(); "
        "print('PRODUCT', any(m.startswith('paper_2407_17678_b200') for m in sys.modules), "
        "'libs2attn' in maps, 'libshardattn_b200' in maps)" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    last = [ln for ln in r.stdout.splitlines() if ln.startswith("PRODUCT")][-1]
    assert last == "PRODUCT False False False", last
