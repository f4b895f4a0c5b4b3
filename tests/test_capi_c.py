"""The C-ABI from plain C (tests/c/capi_demo.c, no Python in the caller):
it compiles against include/tal_b200.h and links libtal_b200.so on any host;
on a GPU its tal_assemble and tal_assemble_elements results match the oracle."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2403_08777_b200"


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    if not (PKG / "libtal_b200.so").exists():
        from paper_2403_08777_b200 import build
        build.build()
    exe = tmp_path_factory.mktemp("capi") / "capi_demo"
    subprocess.run(["gcc", "-O2", "-std=c11", "-I", str(ROOT / "include"), str(ROOT / "tests/c/capi_demo.c"),
                    "-o", str(exe), "-L", str(PKG), "-l:libtal_b200.so", f"-Wl,-rpath,{PKG}", "-lm"],
                   check=True)
    return exe


def test_c_caller_links_and_reports_abi(demo):
    from paper_2403_08777_b200 import _native as N
    out = subprocess.run([str(demo), "--abi"], capture_output=True, text=True, check=True).stdout
    assert int(out) == N.lib().tal_abi_version()


@pytest.mark.gpu
def test_c_caller_assembles_like_the_oracle(demo, tmp_path, oracle):
    import paper_2403_08777_b200 as tb
    nx, ny, nz = 9, 8, 7
    f = tmp_path / "out.bin"
    r = subprocess.run([str(demo), str(nx), str(ny), str(nz), str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    m = tb.generate_box_mesh(nx, ny, nz)
    d = np.fromfile(f, dtype=np.float64).reshape(3, m.n_nodes, 3)
    u, rhs, rhs_seam = d
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u)
    scale = np.abs(ref).max()
    assert np.abs(rhs - ref).max() <= 1e-12 * scale
    assert np.abs(rhs_seam - ref).max() <= 1e-12 * scale
