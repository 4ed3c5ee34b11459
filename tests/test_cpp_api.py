"""The C++ host API (include/sptrain/b200.hpp) compiled with g++ against libsptrain_b200.so: host logic and
error mapping on CPU; a tiny layer step on the GPU (pytest -m gpu).  When the reference's headers are present
(this container only), the same program is also compiled against the reference's own sptrain/errors.hpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2506_13996_b200")
REF_INC = "/root/reference/proj/include"


def _build(out, extra=()):
    src = os.path.join(ROOT, "tests", "cpp", "api_test.cpp")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), *extra, src, "-o", out, "-L", LIBDIR,
           "-lsptrain_b200", f"-Wl,-rpath,{LIBDIR}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_cpp_api_host_logic(tmp_path):
    exe = _build(str(tmp_path / "api_test"))
    r = subprocess.run([exe, "--cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_cpp_api_builds_against_reference_errors(tmp_path):
    exe = _build(str(tmp_path / "api_test_ref"), ("-I", REF_INC))
    r = subprocess.run([exe, "--cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "reference sptrain/errors.hpp" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_layer_step_gpu(tmp_path):
    exe = _build(str(tmp_path / "api_test_gpu"))
    r = subprocess.run([exe, "--gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
