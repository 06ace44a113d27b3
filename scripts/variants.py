"""Build library variants with -D overrides (tuning experiments; product path uses the default build)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12511_b200 import build as b
for spec in sys.argv[1:]:
    name, _, defs = spec.partition(':')
    d = dict(kv.split('=') for kv in defs.split(',') if kv)
    print(b.build_variant(name, d))
