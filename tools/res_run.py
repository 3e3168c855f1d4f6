import sys, os
sys.path.insert(0, os.getcwd())
from paper_2110_13368_b200 import workloads as W
w = W.CONFIGS[sys.argv[1]](int(sys.argv[2]))
s = W.session_for(w)
s.advance(int(sys.argv[2]), w.dt)
s.synchronize()
s.close()
