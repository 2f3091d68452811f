"""Count sequential fallbacks of the speculative reconstruction (workspace word 2)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0712_4046_b200 as k
from bench import CONFIGS, make_inputs
for cname in ("c2", "c1", "c4"):
    cfg = CONFIGS[cname]
    f, g = make_inputs(cfg)
    for v in (2, 4):
        kb = k.KsBatch(v, cfg["batch"], cfg["n"], cfg["n"], cfg["b"], signed=cfg["signed"])
        fd = torch.from_numpy(f.view(np.int32)).cuda(); gd = torch.from_numpy(g.view(np.int32)).cuda()
        kb(fd, gd); kb.status()
        w = kb.workspace[:12].cpu().numpy().view(np.uint32)
        print(cname, "ks%d" % v, "fallbacks", int(w[2]), "of", cfg["batch"] * (2 if v == 4 else 1), flush=True)
