"""The device generator of the synthetic config volumes (csrc/synth.cu) and
its CPU twin (oracle/synth_ref.c, used by the bench's reference arm so that
arm never loads the product library) produce the same bytes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 0x1806_08741
CASES = [
    (1, (512, 512), np.uint8, 3, [(0, 1)]),
    (2, (2048, 1216), np.float32, 3, [(0, 1)]),
    (3, (1024, 1024, 1024), np.uint16, 1, [(0, 3), (511, 514), (1021, 1024)]),
    (4, (512, 512, 256), np.float32, 4, [(0, 4), (130, 133), (252, 256)]),
    (5, (2048, 1216, 7000), np.uint8, 3, [(0, 2), (3500, 3502), (6997, 7000)]),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"config{c[0]}")
def test_device_generator_equals_cpu_twin(sslic, oracle_lib, case):
    import torch
    cfg, dims, dtype, ch, ranges = case
    tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32}[dtype]
    plane = int(np.prod(dims[:2]))
    for z0, z1 in ranges:
        buf = torch.empty(plane * (z1 - z0) * ch, dtype=tdt, device="cuda")
        sslic.synth_generate(cfg, dims, dtype, ch, SEED, z0, z1, buf.data_ptr())
        torch.cuda.synchronize()
        dev = buf.cpu().numpy().view(dtype)
        host = oracle_lib.synth_generate(cfg, dims, dtype, ch, SEED, z0, z1)
        assert dev.tobytes() == host.tobytes(), (
            f"config {cfg} planes [{z0},{z1}): {int((dev != host).sum())} values differ")
