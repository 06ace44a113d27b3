"""Path coverage: test builds of libpbng with small tier constants, run against the oracle
in a subprocess (tests/variant_runner.py), with assertions that every aggregation path of
the product kernels actually ran (implementation counters in pbng_stats):
  * tier-1 hash: starts split into id-window groups (impl_hash[1]) and starts passed on to
    the bitmap tier (impl_hash[3]);
  * tier-2 bitmap windows (impl[0]), repeat-table overflow -> dense recount (impl[1]),
    dense windows (impl[2]).
The product build uses the same source with larger constants."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SMALL = {"PBNG_HASH_SLOTS": 768, "PBNG_HASH_MAX_PB": "(1u<<14)", "PBNG_WIN_LOG_IDS": 15,
         "PBNG_WIN_LOG_DUP": 9, "PBNG_DENSE_ENTRIES": 4096}


def _run(name, defines):
    sys.path.insert(0, ROOT)
    from paper_2110_12511_b200 import build as b
    lib = b.build_variant(name, defines)
    env = dict(os.environ, PBNG_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "variant_runner.py")], env=env,
                         capture_output=True, text=True, timeout=1800)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_small_tables_every_path(cuda_ok):
    tot = _run("small", SMALL)
    impl, hsh = tot["impl"], tot["impl_hash"]
    assert hsh[0] > 0 and hsh[1] > 0 and hsh[2] > hsh[1] and hsh[3] > 0, hsh
    assert impl[0] > 0 and impl[1] > 0 and impl[2] > 0, impl
