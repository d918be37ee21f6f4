"""Strip timing of the chain CTA's K2 (step 6 of an executor evaluation) in a library built with
EXAGEO_EXTRA_NVCC_FLAGS=-DEXAGEO_POTRF_TRACE (development aid). Usage: chain_k2_trace.py [n] [lib]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_02835_b200 as ex  # noqa: E402
import synth_inputs as si  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
x, y = ex.gen_locations(n, 1)
z = si.normals(n, 2)
X, Y, Z = (torch.from_numpy(a).cuda() for a in (x, y, z))
with ex.Context(device=0, tile_tasks=1, graphs=-1) as c:
    for _ in range(3):
        r = c.loglik_dev(X, Y, Z, (1.0, 0.1, 0.5))
    lib = ctypes.CDLL(os.path.join(os.path.dirname(ex.__file__), "_lib", "libexageo.so"))
    buf = (ctypes.c_longlong * 80)()
    assert lib.exageo_dbg_chain_potrf_trace(buf) == 0
    t = list(buf)
    print(f"n={n} device {1e3 * r.info['ms_total']:.1f} us")
    print("chain K2 step 6 (cycles from body start): load %d strips %d %d %d %d  W done %d  end %d"
          % tuple(t[i] - t[0] for i in range(1, 8)))
    print("K0 cycles per pivot:", " ".join(str(v) for v in t[32:48]))
    c = t[64:72]
    print("chain TRSM/SYRK of step 6 (cycles from the body's end): staged %d, mma (warp 0) %d, barrier %d, "
          "stored+barrier %d | SYRK staged %d, mma+barrier %d, stored+barrier %d"
          % tuple(v - c[0] for v in c[1:8]))
