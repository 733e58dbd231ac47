"""The multi-rank NCCL code path of libpm4g (A11 C1 / C2, NEXT-2 min / max,
NEXT-3 EFG limbs, NEXT-4 repartition) run for real with R ranks as threads on
one GPU, through a loopback NCCL (tests/fake_nccl/fake_nccl.cpp) loaded via
PM4G_NCCL_LIB -- NCCL itself refuses two ranks on one device.  Runs in a
subprocess so the loopback library never meets the real NCCL."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fake_nccl")


@pytest.fixture(scope="module")
def fake_lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("fake_nccl") / "libfakenccl.so")
    subprocess.check_call(["nvcc", "-O1", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                           os.path.join(HERE, "fake_nccl.cpp"), "-o", out])
    return out


@pytest.mark.parametrize("R,name", [(2, "tiny"), (3, "tiny"), (2, "bpic2019")])
def test_multi_rank_paths_through_loopback_nccl(fake_lib, R, name):
    env = dict(os.environ, PM4G_NCCL_LIB=fake_lib)
    p = subprocess.run([sys.executable, os.path.join(HERE, "run_ranks.py"), str(R), name], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and f"OK {R}" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]
