"""Config 3: 16 orbit views per step through MultiViewRenderer with 1 / 2 / 3 contexts in flight."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import RenderOptions
from paper_2412_11752_b200.parallel import MultiViewRenderer
sc = scenes.config_scene(3)
cams = scenes.config_cameras(3)[:16]
raw = torch.from_numpy(sc.f32()).cuda()
opt = RenderOptions(sh_degree=3)
for inflight in (1, 2, 3, 2):
    mv = MultiViewRenderer(0, inflight)
    for _ in range(2):
        mv.render(raw, cams, opt)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); mv.render(raw, cams, opt); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    mp = 16 * 1920 * 1080 / 1e6
    print(f"inflight {inflight}: {[round(t, 1) for t in ts]} ms per 16 views -> {mp / (min(ts) * 1e-3):.1f} MP/s (best), "
          f"{mp / (sum(ts) / len(ts) * 1e-3):.1f} MP/s (mean); mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
    mv.close()
