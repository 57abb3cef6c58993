"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/sslic_b200.h declares, and the Python mirror's
host-side validation matches the reference's exception classes
(slic.hpp:52-64, image.hpp:238-249). No compute call is made here."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sslic_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sslic_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_1806_08741_b200 as s
    lib = ctypes.CDLL(s.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [n for n in syms if not hasattr(lib, n)]
    assert not missing, missing


def test_python_mirror_binds_every_symbol():
    import paper_1806_08741_b200 as s
    L = s.lib()
    for n in declared_symbols():
        assert getattr(L, n).restype is not None or n.endswith("destroy"), n


def test_host_validation_mirrors_reference_exceptions():
    import paper_1806_08741_b200 as s
    with pytest.raises(s.InvalidArgument):
        s.NDImage((0, 4), 1, [])
    with pytest.raises(s.InvalidArgument):
        s.NDImage((2, 2), 1, [0.0, 1.0, np.nan, 2.0])
    with pytest.raises(s.InvalidArgument):
        s.NDImage((2, 2, 2, 2, 2), 1, np.zeros(32))
    with pytest.raises(s.InvalidArgument):
        s.SlicParams(grid=[9, 8]).validate((8, 8))
    with pytest.raises(s.InvalidArgument):
        s.SlicParams(grid=[4]).validate((8, 8))
    with pytest.raises(s.InvalidArgument):
        s.SlicParams(grid=[4, 4], weight_m=-1).validate((8, 8))
    assert s.SlicParams(grid=[4, 4]).iterations_for(2) == 10
    assert s.SlicParams(grid=[4, 4, 4]).iterations_for(3) == 5
    assert s.SlicParams(grid=[4], max_iterations=3).iterations_for(3) == 3
    assert s.size_threshold([10, 10]) == 25 and s.size_threshold([5, 4, 3]) == 15
    assert s.cluster_count((100, 100), (50, 50)) == 4
    assert s.cluster_count((2048, 1216, 7000), (32, 32, 32)) == 532608


def test_no_cpu_fallback_without_device():
    """On a machine without a CUDA device every compute entry point fails
    loudly instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_1806_08741_b200 as s
    with pytest.raises(s.CudaError):
        s.run_slic(s.NDImage.zeros((8, 8), 1), s.SlicParams(grid=[4, 4]))


def test_library_holds_sm100a_kernels_only():
    """The product library is built for sm_100a alone (no other targets, no
    PTX-JIT fallback) and holds the hot kernels: the general and the
    first-iteration variants of k_assign_fast / k_assign_lean, the fused
    update and the connectivity kernels (cuobjdump, no GPU needed)."""
    import shutil
    import subprocess
    import paper_1806_08741_b200 as s
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-lelf", s.LIB_PATH], capture_output=True, text=True).stdout
    elfs = [l for l in out.splitlines() if ".cubin" in l]
    assert elfs and all("sm_100a" in l for l in elfs), elfs[:4]
    ptx = subprocess.run([tool, "-lptx", s.LIB_PATH], capture_output=True, text=True).stdout
    assert ".ptx" not in ptx or "sm_100a" in ptx
    syms = subprocess.run(["nm", "-C", s.LIB_PATH], capture_output=True, text=True).stdout
    for kernel in ("k_assign_fast<3, 1, unsigned short, 32, 16, 16, 0, 3>",   # config 3, general
                   "k_assign_fast<3, 1, unsigned short, 32, 16, 16, 0, 7>",   # config 3, iteration 0
                   "k_assign_fast<3, 4, float, 16, 16, 8, 0, 34>",            # config 4
                   "k_assign_lean<3, unsigned char, 32, 32, 32, 40, 4, 0>",   # config 5
                   "k_assign_lean<3, unsigned char, 32, 32, 32, 40, 4, 1>",
                   "k_update_fused", "k_init_perturb", "k_region_cand<3>"):
        assert kernel in syms, kernel
