"""Each step op alone after a clean L2 flush (bench.DeviceStep.isolated_us) under FP8FLOW_* knob
settings given as arguments, e.g.  python tools/time_ops_isolated.py CTAS_PER_SM_A3=2 CTAS_PER_SM_A3=4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
hw = bench.HostWorkload(0)
ds = bench.DeviceStep(hw, dev)
ds.launch_ops(record=False)
torch.cuda.synchronize()
ref = ds.checksums()
for setting in sys.argv[1:] or [""]:
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=")
        os.environ["FP8FLOW_" + k] = v
    iso = ds.isolated_us()
    ds.launch_ops(record=False)
    torch.cuda.synchronize()
    print(f"[{setting}] " + "  ".join(f"{k} {v:.1f}" for k, v in iso.items()) + f"  outputs unchanged: {ds.checksums() == ref}",
          flush=True)
