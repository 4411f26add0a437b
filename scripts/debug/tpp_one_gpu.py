"""Does running the T stages on separate streams of ONE GPU (threaded TPP,
blocks pipelined) beat the sequential engine at the 14B shape?  Steady FPS
from the decode spacing of the last blocks."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2512_04677_b200 as lp
from paper_2512_04677_b200.model import WAN_14B

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for mode in ("sequential", "tpp"):
    cfg = lp.EngineConfig(mode=mode, profile=WAN_14B, precision="bf16", steps=4, cache_capacity=4, blocks=blocks,
                          device_inputs=True, devices=(0,))
    t0 = time.perf_counter()
    res = lp.run(cfg)
    dt = time.perf_counter() - t0
    dec = sorted([e for e in res.timeline if e.kind == "decode"], key=lambda e: e.block)
    sp = [(dec[i].end - dec[i - 1].end) for i in range(len(dec) - 4, len(dec))]
    print(f"{mode}: wall {dt:.1f}s for {blocks} blocks; last decode spacings ms {[round(1e3 * s, 1) for s in sp]}; "
          f"steady FPS {12 / (sum(sp) / len(sp)):.2f}", flush=True)
