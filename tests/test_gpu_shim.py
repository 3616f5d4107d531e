"""C++ drop-in: compile tests/cpp/test_shim.cpp against libshardattn_b200.so
(the reference's shardattn:: API over the B200 kernels) and run it."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _build(tmp_path):
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"])
    pkg = os.path.join(ROOT, "paper_2407_17678_b200")
    olib = os.path.join(ROOT, "oracle", "lib")
    exe = str(tmp_path / "test_shim")
    subprocess.check_call([
        "g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include", "shardattn_b200"),
        "-I", os.path.join(ROOT, "include"), os.path.join(HERE, "cpp", "test_shim.cpp"), "-o", exe,
        f"-L{pkg}", "-lshardattn_b200", f"-L{olib}", "-ls2oracle", f"-Wl,-rpath,{pkg}:{olib}"])
    return exe


def test_shim_builds_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_shim_reference_tests_pass_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr


def test_shim_serialize_and_analysis(tmp_path):
    """Host-only half of the drop-in: serialize.hpp / analysis.hpp through
    libshardattn_b200.so (restates test_serialize.cpp / test_analysis.cpp)."""
    pkg = os.path.join(ROOT, "paper_2407_17678_b200")
    json_dir = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
    exe = str(tmp_path / "test_shim_serialize")
    subprocess.check_call([
        "g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include", "shardattn_b200"),
        "-I", os.path.join(ROOT, "include"), "-I", json_dir,
        os.path.join(HERE, "cpp", "test_shim_serialize.cpp"), "-o", exe,
        f"-L{pkg}", "-lshardattn_b200", "-ls2attn", f"-Wl,-rpath,{pkg}"])
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
