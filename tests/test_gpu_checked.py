"""Device-side checking (VERDICT r1 "race/sync checking"; compute-sanitizer is
closed on the GPU pool): the checked build lib/libhq_check.so
(-DHQ_DEVICE_CHECKS) puts a watchdog on every mbarrier wait of the
tensor-core pipelines (a phase that never completes -- a missing arrive, a
wrong parity, an expect-tx count that never lands -- traps instead of
hanging) and bounds checks on every bulk-copy source and global store of the
tensor-core and SIMT kernels.  The sanitizer workload (every kernel family,
the 12q compiled circuit, a virtual-shard circuit with folded packs) must run
clean and match the oracle under it."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_clean():
    sys.path.insert(0, ROOT)
    from paper_2111_06868_b200 import build
    lib = build.build(checked=True)
    env = dict(os.environ, HQ_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "checked_run.log"), "w") as f:
        f.write(out)
    assert r.returncode == 0, out[-3000:]
    assert "SANITIZE_RUN_OK" in out and "hq device check" not in out, out[-3000:]
