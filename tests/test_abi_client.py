"""The C ABI used from plain C (tests/abi_client.c): no Python or torch on
the library's side of the boundary, only cudart and libmfg_b200.so, as a
reference-side binding would use it. The client checks
mfg_omega_build / mfg_layout_build / mfg_sweep / mfg_sweep_host against a
direct host computation (fp64, 1e-11) and the error path of mfg_sweep."""

import os
import shutil
import subprocess

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def test_pure_c_client(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    libdir = os.path.join(REPO, "paper_2204_14067_b200")
    exe = str(tmp_path / "abi_client")
    subprocess.run([cc, "-O2", "-std=c11", os.path.join(REPO, "tests", "abi_client.c"),
                    "-I", os.path.join(cuda, "include"), "-L", os.path.join(cuda, "lib64"),
                    "-L", libdir, "-lmfg_b200", "-lcudart", "-lm",
                    f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", exe],
                   check=True)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "abi client ok" in res.stdout
