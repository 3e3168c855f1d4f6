"""Phase timeline of the plane-cluster x+y kernel (design tool).

Needs the variant library built with -DBIODIFF_XYC_TRACE:
    make -C paper_2110_13368_b200 OBJ=$PWD/paper_2110_13368_b200/_build_tr/ \
        LIB=$PWD/paper_2110_13368_b200/_lib/libbiodiff_b200_tr.so NVCCFLAGS="... -DBIODIFF_XYC_TRACE"
    BIODIFF_LIB=libbiodiff_b200_tr.so python tools/xyc_trace_probe.py

Prints, per plane round, the x-phase, barrier-wait and y-phase durations
(globaltimer, ns) over the 32 warps of each cluster.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    os.environ.setdefault("BIODIFF_XY_FUSED", "2")
    import paper_2110_13368_b200 as B
    from paper_2110_13368_b200 import workloads as W
    w = W.make("probe", (256, 256, 256), 4, 0, 5)
    s = W.session_for(w)
    s.advance(5, w.dt, with_sources=False)
    s.synchronize()
    s.diffuse_decay_step()
    s.synchronize()
    n = 4096 * 32 * 4
    buf = (ctypes.c_ulonglong * n)()
    rc = B.lib().biodiff_debug_xyc_trace(buf, ctypes.c_longlong(n))
    assert rc == 0, rc
    t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 32, 4)[:256].astype(np.int64)
    t0 = t[:, :, 0].min()
    t = t - t0
    x = t[:, :, 1] - t[:, :, 0]
    bw = t[:, :, 2] - t[:, :, 1]
    y = t[:, :, 3] - t[:, :, 2]
    print("kernel span us: %.1f" % (t[:, :, 3].max() / 1e3))
    print("per-warp item us: x mean %.2f max %.2f | barrier wait mean %.2f | y mean %.2f max %.2f" %
          (x.mean() / 1e3, x.max() / 1e3, bw.mean() / 1e3, y.mean() / 1e3, y.max() / 1e3))
    # per plane: x phase span (first x start -> last x end), y span
    xs = (t[:, :, 1].max(1) - t[:, :, 0].min(1)) / 1e3
    ys = (t[:, :, 3].max(1) - t[:, :, 2].min(1)) / 1e3
    print("per-plane x span mean %.2f, y span mean %.2f us" % (xs.mean(), ys.mean()))
    for P in list(range(0, 3)) + list(range(37, 40)) + [100, 200, 250]:
        print("plane %3d: x start %7.2f end(max) %7.2f | y start %7.2f end(max) %7.2f | x item min/med/max %.2f/%.2f/%.2f y %.2f/%.2f/%.2f" % (
            P, t[P, :, 0].min() / 1e3, t[P, :, 1].max() / 1e3, t[P, :, 2].min() / 1e3, t[P, :, 3].max() / 1e3,
            x[P].min() / 1e3, np.median(x[P]) / 1e3, x[P].max() / 1e3, y[P].min() / 1e3, np.median(y[P]) / 1e3,
            y[P].max() / 1e3))
    hist = np.histogram(t[:, :, 0].min(1) / 1e3, bins=10)
    print("plane start histogram:", hist[0].tolist(), [round(v, 1) for v in hist[1].tolist()])
    s.close()


if __name__ == "__main__":
    main()
