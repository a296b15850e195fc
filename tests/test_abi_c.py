"""The C ABI from a plain C99 client (examples/c_api_example.c): the header is
valid C, every declared symbol links, and argument errors come back as status
codes with messages.  Runs on the CPU-only build host (tf_init then reports the
missing device instead of aborting)."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT


def test_c_client_compiles_links_and_runs(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    lib = os.path.join(ROOT, "paper_1502_05216_b200", "lib")
    if not os.path.exists(os.path.join(lib, "libtwofold_b200.so")):
        pytest.skip("library not built")
    exe = tmp_path / "tf_example"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_api_example.c"), "-L", lib,
                    "-ltwofold_b200", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True,
                         env={**os.environ, "LD_LIBRARY_PATH": lib}, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "ABI version 1" in out.stdout
    assert "negative count -> -1" in out.stdout
    assert "unknown function -> -1" in out.stdout
    assert "empty t_add -> 0" in out.stdout


@pytest.mark.gpu
def test_c_client_host_arrays(tmp_path, cuda):
    """The same C99 client on a GPU box: tf_eval_host on plain host arrays."""
    lib = os.path.join(ROOT, "paper_1502_05216_b200", "lib")
    exe = tmp_path / "tf_example"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_api_example.c"), "-L", lib,
                    "-ltwofold_b200", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True,
                         env={**os.environ, "LD_LIBRARY_PATH": lib}, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "host texp(1) = 0x1.5bf0a8b145769p+1" in out.stdout          # RN(e)
    assert "host tlog1p(1) = 0x1.62e42fefa39efp-1" in out.stdout        # RN(ln 2)


@pytest.mark.gpu
def test_c_client_on_device(tmp_path, cuda):
    lib = os.path.join(ROOT, "paper_1502_05216_b200", "lib")
    exe = tmp_path / "tf_texp"
    cuda_home = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(cuda_home, "include"),
                    os.path.join(ROOT, "examples", "c_texp_device.c"), "-L", lib,
                    "-ltwofold_b200", "-L", os.path.join(cuda_home, "lib64"), "-lcudart",
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True,
                         env={**os.environ, "LD_LIBRARY_PATH": lib + ":" +
                              os.path.join(cuda_home, "lib64")}, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "texp(1) = 0x1.5bf0a8b145769p+1" in out.stdout          # RN(e)
    assert "tlog1p(1) = 0x1.62e42fefa39efp-1" in out.stdout        # RN(ln 2)
