"""Checked build: every entry point and option family on small graphs with the device
checks on (PBNG_CHECK=1, PBNG_DCHECK in device_common.cuh) and small tier constants
(so that every aggregation path fires), each result compared with the oracle
(scripts/sanitize_run.py).  compute-sanitizer is not available on the GPU pool, so the
in-kernel checks of shared-memory table / bitmap indices, emitted partner ids, list
bounds and probe counts stand in for memcheck; a failed check turns the call into
PBNG_ERR_CUDA with the kernel source line."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHECKED = {"PBNG_CHECK": 1, "PBNG_HASH_SLOTS": 768, "PBNG_HASH_MAX_PB": "(1u<<14)", "PBNG_WIN_LOG_IDS": 15,
           "PBNG_WIN_LOG_DUP": 9, "PBNG_DENSE_ENTRIES": 4096}


@pytest.mark.parametrize("name,defines", [("checked", CHECKED), ("checked_prod", {"PBNG_CHECK": 1})])
def test_checked_build(cuda_ok, name, defines):
    sys.path.insert(0, ROOT)
    from paper_2110_12511_b200 import build as b
    lib = b.build_variant(name, defines)
    env = dict(os.environ, PBNG_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_run.py")], env=env,
                         capture_output=True, text=True, timeout=1800)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
