import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions, FrameGrad
r = Rasterizer(0)
sc = scenes.random_scene(int(__import__("os").environ.get("NP", "2000")), seed=29, sh_degree=3, clusters=12)
cam = scenes.look_at_camera(int(__import__("os").environ.get("W", "64")), int(__import__("os").environ.get("H", "48")), (0.3, 0.2, -3.2))
raw = torch.from_numpy(sc.f32()).cuda()
dcol = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, (cam.height, cam.width, 3)).astype(np.float32)).cuda()
for rk in [int(a) for a in sys.argv[1:]]:
    fb = r.render(raw, cam, RenderOptions(sh_degree=3, raster_kernel=rk))
    g = r.backward_render(raw, FrameGrad(d_color=dcol))
    torch.cuda.synchronize()
    print(rk, 'ok', float(g.raw.norm()), flush=True)
