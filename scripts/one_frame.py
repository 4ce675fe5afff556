"""One forward (and optionally backward) of a BASELINE config: the short command
profiled under ncu.  usage: python scripts/one_frame.py CFG [bwd] [repeats]"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import FrameGrad, Rasterizer, RenderOptions

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
bwd = len(sys.argv) > 2 and sys.argv[2] == 'bwd'
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
r = Rasterizer(0)
sc = scenes.config_scene(cfg)
cam = scenes.config_cameras(cfg)[0]
raw = torch.from_numpy(sc.f32()).cuda()
opt = RenderOptions(sh_degree=scenes.CONFIGS[cfg]['sh_degree'])
for _ in range(reps):
    fb = r.render(raw, cam, opt)
    if bwd:
        tgt = torch.from_numpy(scenes.config_target(cfg, cam).astype(np.float32)).cuda()
        v, d = r.l1_loss(fb.color, tgt)
        g = r.backward_render(raw, FrameGrad(d_color=d))
torch.cuda.synchronize()
print('ok', cfg, 'bwd' if bwd else 'fwd', r.stats()['pairs'])
