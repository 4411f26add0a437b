import sys, os, time, threading
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2512_04677_b200 as lp
from paper_2512_04677_b200 import _lib as L
L.init_device(0)
# 1. raw link ping between two streams
abort = torch.zeros(4, dtype=torch.int32, device="cuda:0")
from paper_2512_04677_b200.engine import DeviceLink
link = DeviceLink(192, 1, 0, abort, 5.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
src = torch.arange(48, dtype=torch.float32, device="cuda:0")
dst = torch.zeros(48, device="cuda:0")
status = torch.full((1,), -1, dtype=torch.int32, device="cuda:0")
link.recv(dst, s2, 0, status)
link.send(src, s1, 0)
torch.cuda.synchronize()
print("ping ok", torch.equal(src, dst), status.item(), link.flags.tolist())
for graphs in (False, True):
    t0 = time.time()
    try:
        r = lp.run_tpp(lp.EngineConfig(mode="tpp", steps=4, blocks=3, use_graphs=graphs, link_timeout_s=5.0))
        s = lp.run_sequential(lp.EngineConfig(mode="sequential", steps=4, blocks=3))
        print("graphs", graphs, "ok", time.time() - t0, all(a.values.tobytes() == b.values.tobytes() for a, b in zip(r.blocks, s.blocks)))
    except Exception as e:
        print("graphs", graphs, "FAILED", time.time() - t0, repr(e)[:300])
