"""Reference-precision forward (fp64_alpha) of config 2: time and framebuffer digest."""
import hashlib, os, sys, time
import torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions
r = Rasterizer(0)
sc = scenes.config_scene(2)
cam = scenes.config_cameras(2)[0]
raw = torch.from_numpy(sc.f32()).cuda()
opt = RenderOptions(sh_degree=3, fp64_alpha=True)
for _ in range(2):
    fb = r.render(raw, cam, opt)
torch.cuda.synchronize(); t = time.time()
for _ in range(3):
    fb = r.render(raw, cam, opt)
torch.cuda.synchronize(); dt = (time.time() - t) / 3
h = hashlib.sha1(b''.join(getattr(fb, f).cpu().numpy().tobytes() for f in ('color', 'depth', 'normal', 'alpha')))
print(f"fp64_alpha forward mode={os.environ.get('DRK_FP64_ALL', 'warp')}: {dt*1e3:.1f} ms digest {h.hexdigest()[:16]}", flush=True)
