"""Run one KS shape through every variant with a sync and error check after each
(debug helper).  usage: repro_case.py n b [batch]"""
import sys, random
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0712_4046_b200 as k
from paper_0712_4046_b200.words import ints_to_words, words_to_ints
from oracle import ks_oracle as O
n, b = int(sys.argv[1]), int(sys.argv[2]); B = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rng = random.Random(n * 1000 + b)
fs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
gs = [[rng.randrange(1 << b) for _ in range(n)] for _ in range(B)]
w = (b + 31) // 32
fd = torch.from_numpy(np.stack([ints_to_words(f, w) for f in fs]).view(np.int32)).cuda()
gd = torch.from_numpy(np.stack([ints_to_words(g, w) for g in gs]).view(np.int32)).cuda()
want = [O.ks_mul(1, fs[p], gs[p], b, mode="native") for p in range(B)]
for v in (1, 2, 3, 4):
    for seq in (0,):
        try:
            kb = k.KsBatch(v, B, n, n, b)
            h = kb(fd, gd)
            torch.cuda.synchronize()
            kb.status()
            got = [words_to_ints(h[p].cpu().numpy().view(np.uint32)) for p in range(B)]
            print(v, "ok" if got == want else "MISMATCH", flush=True)
        except Exception as e:
            print(v, "ERROR", repr(e), flush=True)
            raise
