"""GPU test of the C++ host layer (paper_2011_09017_b200/cpp/acz_b200.hpp): the compiled
test program exercises the reference-signature codec, error mapping, device path and the
adaptive controller; its ACZ1 output must equal the oracle's bytes."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_cpp_host_layer(gpu_lib, oracle, tmp_path):
    from paper_2011_09017_b200 import build as B
    exe = B.build_cpp_test()
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    x = np.fromfile(tmp_path / "host.f32", dtype=np.float32).reshape(4, 16, 56, 56)
    blob = (tmp_path / "host.acz1").read_bytes()
    assert blob == oracle.compress(x, 1e-3).blob
