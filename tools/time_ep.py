"""NEXT-3 timing alone (bench.py's ep_measure): python tools/time_ep.py [reps]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2511_02302_b200 import roofline as RL  # noqa: E402

if __name__ == "__main__":
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    peak = RL.measured_peaks(bench.ROOT)["hbm_gbs"]
    print(json.dumps(bench.ep_measure(torch.device("cuda", 0), peak, reps), indent=1))
