import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 and the sm_100a library")
    config.addinivalue_line(
        "markers", "slow: long CPU oracle runs")
