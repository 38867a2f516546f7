"""The proj/core drop-in (BASELINE north_star): the reference's own core
library with src/codec.cpp replaced by paper_2011_09017_b200/proj_core/gpu_codec.cpp over
libacz_gpu.so, everything else (controller.cpp, huffman.cpp, config.cpp, tensor_io.cpp and
the headers) compiled unmodified (oracle/Makefile `dropin`).

tests/cpp/dropin_controller.cpp drives the reference's acz::Controller
(begin_iteration -> wrap_forward -> unwrap_backward -> collect_stats -> finalize,
src/controller.cpp:124-253) and prints every observable: the GPU build's output must equal
the CPU build's byte for byte (ACZ1 blobs, unwrapped tensors, stash accounting, ledger CSV,
blob-file round trips, exception classes)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
CPU = os.path.join(REF, "dropin_cpu")
GPU = os.path.join(REF, "dropin_gpu")


def _need():
    if not (os.path.exists(CPU) and os.path.exists(GPU)):
        pytest.skip("drop-in binaries not built (oracle/Makefile dropin needs /root/reference)")


def test_dropin_binaries_link():
    """CPU-side: the drop-in library resolves every symbol against libacz_gpu.so."""
    _need()
    out = subprocess.run(["ldd", GPU], capture_output=True, text=True, check=True).stdout
    assert "libacz_core_gpu.so" in out and "libacz_gpu.so" in out and "not found" not in out
    syms = subprocess.run(["nm", "-D", "--defined-only",
                           os.path.join(REF, "libacz_core_gpu.so")],
                          capture_output=True, text=True, check=True).stdout
    # the reference's codec API (include/acz/codec.hpp:54-73) + the controller
    for mangled in ("_ZN3acz8compressERKNS_7TensorTIfEERKNS_11CodecParamsE",
                    "_ZN3acz10decompressERKNS_16CompressedTensorEb",
                    "_ZN3acz15blob_from_bytesEPKhm",
                    "_ZN3acz13blob_to_bytesERKNS_16CompressedTensorE",
                    "_ZN3acz10Controller12wrap_forwardEiONS_7TensorTIfEEb",
                    "_ZN3acz10Controller15unwrap_backwardERNS_16ActivationHandleE"):
        assert mangled in syms, mangled


@pytest.mark.gpu
@pytest.mark.parametrize("zr,pred", [("filter", "prev"), ("relu", "prev"),
                                     ("filter", "lorenzo2d"), ("relu", "lorenzo2d")])
def test_reference_controller_over_gpu_codec(zr, pred):
    _need()
    cpu = subprocess.run([CPU, zr, pred], capture_output=True, text=True, timeout=600)
    gpu = subprocess.run([GPU, zr, pred], capture_output=True, text=True, timeout=600)
    assert cpu.returncode == 0, cpu.stderr
    assert gpu.returncode == 0, gpu.stderr
    a, b = cpu.stdout.splitlines(), gpu.stdout.splitlines()
    assert sum(" kind=blob " in line for line in a) >= 20  # the controller really compressed
    for i, (x, y) in enumerate(zip(a, b)):
        assert x == y, f"line {i}:\n cpu: {x}\n gpu: {y}"
    assert len(a) == len(b)
