import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    """A GPU test that hangs (e.g. a device-side wait that never ends) is ended after 300 s by
    pytest-timeout's thread method — it works even when the main thread is blocked inside a
    CUDA call — instead of stalling the whole run."""
    if not config.pluginmanager.hasplugin("timeout"):
        return
    for item in items:
        if item.get_closest_marker("gpu") and not item.get_closest_marker("timeout"):
            item.add_marker(pytest.mark.timeout(300, method="thread"))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test ran without a CUDA device")
    from paper_2502_06766_b200 import _lib

    _lib.load()
    _lib.check(_lib.load().tkv_device_check())
    return torch.device("cuda", 0)


def sample_rows(n: int, seg: int, k: int = 1 << 30) -> np.ndarray:
    """Rows the sampled threshold scores for segment seg = b * Hkv + kv head (restates
    sample_row / sample_stride in paper_2502_06766_b200/csrc/internal.h): adversarial caches put
    their outliers exactly there to force the exactness fallback."""
    target = 2048 if (n <= (1 << 17) and k * 32 <= n) else 4096  # sample_max: half the sample
    stride = max(8, -(-n // target))
    h = (seg * 0x9E3779B9 + 0x7F4A7C15) & 0xFFFFFFFF
    r = np.arange(-(-n // stride), dtype=np.int64) * stride + (h >> 8) % stride
    return np.minimum(r, n - 1)


def bf16_normal(rng: np.random.Generator, shape) -> np.ndarray:
    from oracle.oracle import to_bf16_f32

    return to_bf16_f32(rng.standard_normal(shape, dtype=np.float32))
