"""Time the bench's ensemble extras (C2 3 members, Ensemble-2 / -3) for an A/B run."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_10709_b200 import fin  # noqa: E402

r = bench.ensembles(fin, torch)
print(json.dumps({k: round(v["env_steps_per_s"] / 1e6, 1) for k, v in r.items()}))
