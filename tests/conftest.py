"""pytest configuration: the `gpu` marker and import paths.

`-m "not gpu"` runs here on CPU (oracle pinning, host logic, C-ABI load and
symbol checks, multi-process gloo tests); `-m gpu` runs the parity tests proper
on a B200 through the C-ABI.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); the parity tests proper")
