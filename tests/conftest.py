import pathlib
import sys


ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def golden_layer_cases():
    return sorted(GOLDEN.glob("layer_*.npz"))


def golden_lut_cases():
    return sorted(p for p in GOLDEN.glob("lut_d*_n*.npz"))


def golden_kind_cases():
    """Other basis families (LUT mode) and the exact-evaluation path."""
    return sorted(GOLDEN.glob("kind_*.npz"))


def golden_kind_lut_cases():
    return sorted(GOLDEN.glob("lutk_*.npz"))
