"""The pins catch plausible mistakes: each mutant of tests/_mutants.py plants ONE slip in the oracle
(a dropped factor, a wrong sign or index, a swapped coefficient or operand) and the pin suite
tests/test_oracle_pins.py, run against the mutated oracle, must fail.  A surviving mutant names a
part of the oracle that nothing pins (no GPU; the mutants run in parallel subprocesses)."""
import concurrent.futures as cf
import importlib.util
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
_spec = importlib.util.spec_from_file_location("isrs_oracle_mutants", os.path.join(HERE, "_mutants.py"))
_mut = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mut)
NAMES = sorted(_mut.MUTANTS)


def _run(name):
    env = dict(os.environ, ISRS_ORACLE_MUTANT=name, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1",
               MKL_NUM_THREADS="1")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(HERE, "test_oracle_pins.py"), "-x", "-q",
                        "-p", "no:cacheprovider", "-m", "not gpu"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    return r.returncode, r.stdout[-1500:]


@pytest.fixture(scope="module")
def outcomes():
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        return dict(zip(NAMES, ex.map(_run, NAMES)))


@pytest.mark.parametrize("name", NAMES)
def test_pins_kill_mutant(outcomes, name):
    rc, tail = outcomes[name]
    assert rc == 1, f"mutant {name} survived the pins (pytest rc={rc}):\n{tail}"
