"""Config 3, one context: per-view host checkpoints (DRK_HOST_TRACE) over 3 passes of 16 views."""
import sys, time
import torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions
r = Rasterizer(0)
sc = scenes.config_scene(3)
cams = scenes.config_cameras(3)[:16]
raw = torch.from_numpy(sc.f32()).cuda()
opt = RenderOptions(sh_degree=3)
for c in cams:
    r.render(raw, c, opt)
torch.cuda.synchronize()
print("---- timed passes", file=sys.stderr, flush=True)
for p in range(3):
    t = time.perf_counter()
    for c in cams:
        r.render(raw, c, opt)
    torch.cuda.synchronize()
    print(f"pass {p}: {(time.perf_counter() - t) * 1e3:.0f} ms", file=sys.stderr, flush=True)
