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
