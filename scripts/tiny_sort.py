"""One small merge (16K delta keys, 48-bit values) for ncu launch-list / per-kernel profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.sort_scaling import run
import json
nd = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
print(json.dumps(run(1 << 20, 1 << 16, nd, 0.5, 48, reps=2)))
