"""Config 4 probe: 4M DRK, one 3840x2160 orbit view forward (+ optionally backward); pairs, stage times, memory."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import FrameGrad, Rasterizer, RenderOptions
r = Rasterizer(0)
r.set_timing(True)
t0 = time.time()
sc = scenes.config_scene(4)
cams = scenes.config_cameras(4)
print('scene gen', round(time.time() - t0, 1), 's', flush=True)
raw = torch.from_numpy(sc.f32()).cuda()
opt = RenderOptions(sh_degree=3)
for v in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    torch.cuda.synchronize(); t = time.time()
    fb = r.render(raw, cams[v], opt)
    torch.cuda.synchronize(); dt = time.time() - t
    st = r.stats()
    free, total = torch.cuda.mem_get_info()
    print(f'view {v}: {dt*1e3:.0f} ms pairs {st["pairs"]} fp64px {st["fp64_pixels"]} bands {r.bands()} '
          f'tie runs {st["tie_runs"]} members {st["tie_members"]} max run {st["tie_max_run"]}',
          {k: round(x, 1) for k, x in st['stage_ms'].items()},
          'device mem used GB', round((total - free) / 1e9, 1), flush=True)
    if len(sys.argv) > 2 and sys.argv[2] == 'bwd':
        tgt = torch.from_numpy(scenes.config_target(4, cams[v], view=v).astype(np.float32)).cuda()
        _, d = r.l1_loss(fb.color, tgt)
        torch.cuda.synchronize(); t = time.time()
        g = r.backward_render(raw, FrameGrad(d_color=d))
        torch.cuda.synchronize()
        print(f'  backward {1e3*(time.time()-t):.0f} ms', flush=True)
