"""Phase timing of k_recon_par (debug build tools/libkmx_trace.so, -DKMX_TRACE)."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_0712_4046_b200 import _lib
_lib.LIB_PATH = 'tools/libkmx_trace.so'
import paper_0712_4046_b200 as k
from bench import CONFIGS, make_inputs
L = _lib.lib()
L.kmx_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
for cname, v in (("c2", 4), ("c2", 2), ("c4", 4)):
    cfg = CONFIGS[cname]
    f, g = make_inputs(cfg)
    kb = k.KsBatch(v, cfg["batch"], cfg["n"], cfg["n"], cfg["b"], signed=cfg["signed"])
    fd = torch.from_numpy(f.view(np.int32)).cuda(); gd = torch.from_numpy(g.view(np.int32)).cuda()
    for _ in range(3):
        kb(fd, gd)
    torch.cuda.synchronize()
    L.kmx_prof_enable(1)
    kb(fd, gd)
    ms = (ctypes.c_float * 6)()
    L.kmx_prof_read(ms, 6)
    L.kmx_prof_enable(0)
    t = np.zeros(512, dtype=np.uint64)
    L.kmx_debug_trace(t.ctypes.data, 512)
    t = t.reshape(64, 8).astype(np.int64)
    d = np.diff(t[:, :7], axis=1)
    print(cname, "ks%d" % v, "recon ms", round(ms[3], 4), "phase cycles median (stage, setup, csum+prewalk, exscan, iterations, outwalk, final):",
          [int(x) for x in np.median(d, axis=0)], "start spread", int(t[:, 0].max() - t[:, 0].min()))
