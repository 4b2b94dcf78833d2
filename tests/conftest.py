import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the libmpm CUDA kernels)")
    config.addinivalue_line("markers", "reference: imports the read-only reference package (container only)")


def reference_available() -> bool:
    return (REFERENCE_SRC / "moepipesim" / "__init__.py").exists()


@pytest.fixture(scope="session")
def moepipesim():
    """The unmodified reference package, imported read-only from /root/reference."""
    if not reference_available():
        pytest.skip("reference package not mounted (GPU box); golden fixtures cover this")
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.append(str(REFERENCE_SRC))
    import moepipesim
    return moepipesim


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22175_b200 import _lib
    _lib.load()  # fails loudly if the extension is missing
    return torch.device("cuda", 0)
