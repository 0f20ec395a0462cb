import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle check")
    mutant = os.environ.get("ISRS_ORACLE_MUTANT")
    if mutant:        # tests/test_oracle_mutants.py: plant one slip in the oracle for this session
        import importlib.util
        spec = importlib.util.spec_from_file_location(
            "isrs_oracle_mutants", os.path.join(os.path.dirname(os.path.abspath(__file__)), "_mutants.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.apply(mutant)
