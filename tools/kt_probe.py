"""Per-kernel-class times of a workload's step (kernel timing on: event
pairs per launch, no graph replay). Usage: kt_probe.py c3 [steps]."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2110_13368_b200 import workloads as W

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = W.CONFIGS[name](steps)
s = W.session_for(w)
s.advance(3, w.dt)
s.set_kernel_timing(True)
s.advance(steps, w.dt)
s.synchronize()
t = s.kernel_times()
print(os.environ.get("TAG", ""), " ".join(f"{k}={v[1] / max(v[0], 1) * 1e3:.1f}us" for k, v in t.items() if v[0]))
s.close()
