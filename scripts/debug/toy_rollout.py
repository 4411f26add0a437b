import json, sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2512_04677_b200 as lp
from oracle import livepipe_oracle as O
G = np.load("tests/golden/golden.npz")
def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
cfg = lp.EngineConfig(mode="sequential", steps=4, blocks=3, use_graphs=False)
rt = lp.build_runtime(cfg)
dn = lp.B200Denoiser(rt.weights, rt.schedule, precision="fp32")
caches = {j: lp.RollingKvCache(j, 4) for j in range(1, 5)}
sink = lp.SinkSlot(rt.conditions.reference.copy(), 1)
ob, of, osink = O.run_sequential(O.RolloutCfg(steps=4, blocks=3))
for i in range(3):
    x = lp.noise_block(cfg, i)
    for j in range(4, 0, -1):
        o = dn.denoise_block(x, j, caches[j].view(), lp.BlockCond(rt.conditions.audio_for(i), rt.conditions.prompt), sink.content, i + 1, max_entries=4)
        x = lp.flow_step(x, o.velocity, rt.schedule.dt)
        caches[j].push(o.kv)
    print("dropin block", i, rel(x.values, G["c1_latents"][i]), rel(x.values, ob[i]))
    if i == 0:
        lp.aas_update(sink, x, rt.codec)
        print("sink vs oracle", rel(sink.content, osink))
res = lp.run_sequential(cfg)
print("engine", [rel(b.values, G["c1_latents"][i]) for i, b in enumerate(res.blocks)])
# single-stage debug: step-by-step block 1 via engine stages
