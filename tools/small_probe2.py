"""Sequence probe of the one-cluster kernel (debug tool): runs golden
fixtures through advance() one after another in one process."""
import os, sys
sys.path.insert(0, os.getcwd())
os.environ['BIODIFF_RESIDENT'] = '1'
from tests.test_gpu_parity import load_golden
from tests.helpers import make_session, bits_equal

import glob
names = sys.argv[1:] or sorted(os.path.basename(p)[:-4] for p in glob.glob('tests/golden/*.npz'))
for name in names:
    w, z = load_golden(name)
    if bool(z["initial_clamp"]) or not bool(z["with_sources"]):
        continue
    s = make_session(w)
    s.prepare_advance(w.steps, w.dt, with_sources=True)
    s.advance(w.steps, w.dt, with_sources=True)
    try:
        print(name, w.n, w.S, 'ok', bits_equal(s.download_field(), z['field']), flush=True)
    except Exception as e:
        print(name, w.n, w.S, 'FAIL', e, flush=True)
        break
    s.close()
