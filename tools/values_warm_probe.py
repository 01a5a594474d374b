import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2506_05617_b200 import configs, engine
from paper_2506_05617_b200.pipeline import lfa_device
dev = torch.device("cuda:0")
for cfg in (3, 2):
    layer = configs.WORKLOADS[cfg].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
    for vec, warm in ((False, None), (True, False), (True, True)):
        best = 1e9
        for _ in range(3):
            tm = engine.Timer(dev); tm.mark("a")
            r = lfa_device(w, layer.n, layer.m, "f32", vec, warm_start=warm)
            tm.mark("b"); torch.cuda.synchronize()
            best = min(best, tm.seconds("a", "b"))
        print(f"cfg{cfg} vectors={vec} warm={warm}: {best*1e3:.2f} ms, sweeps {r.info.float().mean().item():.2f}", flush=True)
