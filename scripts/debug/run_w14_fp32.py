"""Debug: the 14B-geometry (2 layers) rollout in fp32 validation mode.
usage: run_w14_fp32.py <blocks> <graphs 0/1> [profile w14|1p3b]"""
import dataclasses
import json
import sys
import time

import torch

import paper_2512_04677_b200 as lp
from oracle import livepipe_oracle as O

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 6
graphs = bool(int(sys.argv[2])) if len(sys.argv) > 2 else True
which = sys.argv[3] if len(sys.argv) > 3 else "w14"
if which == "w14":
    spec = json.load(open("tests/golden/wan_fixtures.json"))["w14_l2"]
    pp = lp.ModelProfile(**dataclasses.asdict(O.wan_profile(**spec["profile"])))
    roll = dict(spec["rollout"], blocks=blocks)
else:
    pp = lp.WAN_1_3B
    if which == "1p3b_l1":
        pp = dataclasses.replace(pp, n_layers=1)
    roll = dict(steps=4, blocks=blocks, cache_capacity=4)
t0 = time.time()
res = lp.run_sequential(lp.EngineConfig(mode="sequential", profile=pp, precision="fp32", use_graphs=graphs, **roll))
torch.cuda.synchronize()
print(which, blocks, "graphs" if graphs else "eager", "ok", round(time.time() - t0, 1), flush=True)
