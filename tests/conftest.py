import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built libkkrx.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionfinish(session, exitstatus):
    """With KK_EQ_PROOF_LOG set, write every eq_check record (frames over the EQ tolerance and the decision
    flips that prove them) as JSON — the evidence that each excused frame is a boundary flip."""
    path = os.environ.get("KK_EQ_PROOF_LOG")
    mod = sys.modules.get("gpu_case")
    if path and mod is not None:
        import json
        with open(path, "w") as f:
            json.dump(mod.PROOFS, f, indent=1)
