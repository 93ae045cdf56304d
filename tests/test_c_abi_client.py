"""A plain-C program built against include/ebc_b200.h and linked with libebc_b200.so (tests/c_abi_client.c):
the drop-in boundary is usable without Python or C++ types.  Without a GPU it must fail loudly with
EBC_ERR_CUDA (there is no CPU fallback); on a GPU it must reproduce the Python mirror's run exactly."""
import os
import subprocess

import numpy as np
import pytest

import paper_1910_11039_b200 as ebc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "_build")
EXE = os.path.join(BUILD, "c_abi_client")


def build_client() -> str:
    ebc.build()
    os.makedirs(BUILD, exist_ok=True)
    libdir = os.path.join(ROOT, "paper_1910_11039_b200")
    subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_abi_client.c"), "-o", EXE, "-L" + libdir, "-lebc_b200",
                    "-Wl,-rpath," + libdir], check=True)
    return EXE


def cuda_present() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_c_client_builds_and_fails_loudly_without_a_gpu():
    exe = build_client()
    if cuda_present():
        pytest.skip("a GPU is present: covered by the gpu test")
    r = subprocess.run([exe, "8", "0.1"], capture_output=True, text=True)
    assert r.returncode == 5                      # EBC_ERR_CUDA
    assert "no CUDA device" in r.stdout and "no CPU fallback" in r.stdout


@pytest.mark.gpu
def test_c_client_matches_python_mirror():
    exe = build_client()
    r = subprocess.run([exe, "12", "0.05"], capture_output=True, text=True, check=True)
    n, m, tau, epochs, checksum = r.stdout.split()
    g = ebc.gen_rmat(12, 16, seed=2).largest_connected_component()
    res, st = ebc.run_pipeline(g, ebc.RunConfig(eps=0.05, delta=0.1, seed=7))
    assert (int(n), int(m)) == (g.num_vertices, g.num_edges)
    assert (int(tau), int(epochs)) == (res.tau_total, st["epochs"])
    assert float(checksum) == pytest.approx(float(np.sum(res.scores)), rel=1e-11)
