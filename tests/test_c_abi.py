"""The C ABI from a plain C program (tests/c/abi_test.c): compiled here with
gcc against include/bspmm.h, linked to libbspmm.so (and liboracle.so as the
reference).  CPU: host-only entry points and argument checks; GPU: a small
batch through offsets, CSR, COO and the host-buffer call, bitwise against O3'."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1903_11409_b200")
ORACLE = os.path.join(ROOT, "oracle")
CUDA = "/usr/local/cuda"


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cabi") / "abi_test")
    cmd = ["gcc", "-std=c11", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "c", "abi_test.c"), "-o", out,
           "-L", LIBDIR, "-lbspmm", "-L", ORACLE, "-loracle", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{LIBDIR}:{ORACLE}:{os.path.join(CUDA, 'lib64')}", "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_c_abi_host_only(exe):
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr


@pytest.mark.gpu
def test_c_abi_gpu(exe):
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
