import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "reference: needs the live reference under /root/reference")


def load_golden(name):
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_rng():
    return load_golden("rng.npz")


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("small_cases.npz")


@pytest.fixture(scope="session")
def golden_powerlaw():
    return load_golden("powerlaw_cases.npz")


@pytest.fixture(scope="session")
def golden_config1():
    return load_golden("config1.npz")


def iter_cases(d):
    """Yield (name, case-dict) for a small/powerlaw golden file."""
    for name in d["names"]:
        name = str(name)
        p = name + "_"
        c = {k[len(p):]: v for k, v in d.items() if k.startswith(p)}
        N, k1, k2, bs = (int(x) for x in c["meta"])
        c.update(N=N, k1=k1, k2=k2, base_seed=bs)
        yield name, c


@pytest.fixture(scope="session")
def reference_fsa():
    """The live reference package (only in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not present (GPU box / fresh checkout)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.append(str(REFERENCE_SRC))
    import fsa  # noqa: F401
    from fsa import kernels
    kernels.warmup(np.float64)
    kernels.warmup(np.float32)
    return fsa


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    oracle.load()
    return oracle
