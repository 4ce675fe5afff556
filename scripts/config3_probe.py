"""Config 3 probe: 1M DRK, first few orbit views at 1080p; pairs, stage times, memory."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions
r = Rasterizer(0)
r.set_timing(True)
t0 = time.time()
sc = scenes.config_scene(3)
cams = scenes.config_cameras(3)
print('scene gen', time.time() - t0, 's', flush=True)
raw = torch.from_numpy(sc.f32()).cuda()
opt = RenderOptions(sh_degree=3)
nv = int(sys.argv[1]) if len(sys.argv) > 1 else 4
for v in range(nv):
    torch.cuda.synchronize(); t = time.time()
    fb = r.render(raw, cams[v], opt)
    torch.cuda.synchronize(); dt = time.time() - t
    st = r.stats()
    print(f'view {v}: {dt*1e3:.1f} ms pairs {st["pairs"]} fp64px {st["fp64_pixels"]}', {k: round(x, 2) for k, x in st['stage_ms'].items()},
          'mem GB', round(torch.cuda.max_memory_allocated() / 1e9, 2), flush=True)
