"""Config 3 views: wall time per view vs the sum of stage times (host gaps)."""
import sys, time
import torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions
r = Rasterizer(0)
sc = scenes.config_scene(3)
cams = scenes.config_cameras(3)[:6]
raw = torch.from_numpy(sc.f32()).cuda()
opt = RenderOptions(sh_degree=3)
for c in cams:
    r.render(raw, c, opt)
torch.cuda.synchronize()
import subprocess
smi = subprocess.Popen(['nvidia-smi', '--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active', '--format=csv,noheader', '-lms', '250'], stdout=open('gpurun_out/mv_clocks.log', 'w'))
for timing in (False, True, False, True):
    r.set_timing(timing)
    for i, c in enumerate(cams):
        torch.cuda.synchronize(); t = time.perf_counter()
        r.render(raw, c, opt)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) * 1e3
        st = r.stats()
        print(f"timing={timing} view {i}: wall {dt:.1f} ms  stages {sum(st['stage_ms'].values()):.1f} ms  pairs {st['pairs']}",
              {k: round(v, 1) for k, v in st['stage_ms'].items() if v}, flush=True)
smi.terminate()
