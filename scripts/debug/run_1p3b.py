"""Run the full 1.3B config through run_sequential in one precision (debug aid)."""
import sys
import time

import torch

import paper_2512_04677_b200 as lp

prec = sys.argv[1]
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 5
t0 = time.time()
res = lp.run_sequential(lp.EngineConfig(mode="sequential", profile=lp.WAN_1_3B, steps=4, blocks=blocks,
                                        cache_capacity=4, precision=prec))
torch.cuda.synchronize()
print(prec, "ok", round(time.time() - t0, 1), "s", [float(abs(b.values).mean()) for b in res.blocks], flush=True)
