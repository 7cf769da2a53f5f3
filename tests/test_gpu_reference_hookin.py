"""The reference's OWN tests run through the device kernels (SURVEY §8(b) "verified hook-in").

``paper_2303_17503_b200.reference_plugin`` re-registers the reference's nine engines with
``core.register(dataclasses.replace(GAME, batch_kernel=K))`` (reference core.py:126-128,
346-348, 366-368, 276-292); the unmodified reference package (baseline/_ref, installed by
tools/install_reference.sh from /root/reference/pkg) then runs its own test files in a subprocess:

* ``test_core.py`` -- batch == scalar fingerprints per game, column agreement, auto-reset, worker
  invariance, offending-slot reporting, observation symmetry (the batch side on the GPU, the
  scalar side on the reference's Python engines);
* ``test_bench.py`` -- BatchSession / bench_run / batch_outputs over the kernels;
* ``test_tictactoe.py`` -- including its numpy-kernel parity test, now against the device kernel;
* ``test_acceptance.py::test_api_contract_auto_reset_per_game`` and ``::test_throughput_scaling``
  (criterion 7: tic-tac-toe 1024/1 >= 4x, >= 7 of 9 games monotone in batch size).

Skipped when baseline/_ref is absent (it is git-ignored; the GPU box gets it with the snapshot).
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "_tests")
SELECTION = [
    "test_core.py",
    "test_bench.py",
    "test_tictactoe.py",
    "test_acceptance.py::test_api_contract_auto_reset_per_game",
    "test_acceptance.py::test_throughput_scaling",
]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "boardbatch")) or not os.path.isdir(TESTS),
                    reason="reference not installed in baseline/_ref (tools/install_reference.sh)")
def test_reference_suite_through_the_device_plugin():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    if env.get("BBK_LIB"):   # the subprocess runs in the reference's test directory
        env["BBK_LIB"] = os.path.join(ROOT, env["BBK_LIB"]) if not os.path.isabs(env["BBK_LIB"]) else env["BBK_LIB"]
    cmd = [sys.executable, "-m", "pytest", "-p", "paper_2303_17503_b200.reference_plugin", "-p", "no:cacheprovider",
           "-q", "-rA", "--rootdir", TESTS] + [os.path.join(TESTS, s) for s in SELECTION]
    r = subprocess.run(cmd, cwd=TESTS, env=env, capture_output=True, text=True, timeout=900)
    log_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(log_dir, exist_ok=True)
    with open(os.path.join(log_dir, "reference_hookin.log"), "w") as fh:
        fh.write(" ".join(cmd) + "\n\n" + r.stdout + "\n" + r.stderr)
    assert "boardbatch B200 plugin: device batch_kernel for" in r.stderr, r.stderr[-3000:]
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-3000:]
