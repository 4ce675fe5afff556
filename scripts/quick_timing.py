"""Quick per-config forward / backward timing (development aid)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions, FrameGrad

r = Rasterizer(0)
r.set_timing(True)
r.set_counters(True)
VALIDATE = '--validate' in sys.argv
sys.argv = [a for a in sys.argv if a != '--validate']
for cfg in [int(a) for a in sys.argv[1:]] or [0, 1, 2]:
    sc = scenes.config_scene(cfg)
    cam = scenes.config_cameras(cfg)[0]
    raw = torch.from_numpy(sc.f32()).cuda()
    opt = RenderOptions(sh_degree=scenes.CONFIGS[cfg]['sh_degree'], raster_kernel=int(os.environ.get('RK', '0')))
    for _ in range(2):
        fb = r.render(raw, cam, opt)
    torch.cuda.synchronize()
    t = time.time(); N = 5
    for _ in range(N):
        fb = r.render(raw, cam, opt)
    torch.cuda.synchronize(); dt = (time.time() - t) / N
    st = r.stats()
    mp = cam.width * cam.height / 1e6
    if VALIDATE:
        r.set_validation(True); r.render(raw, cam, opt); print('validation (max err/bound, max abs err):', r.validation(), r.validation_detail()); r.set_validation(False)
    print(f"cfg{cfg} fwd {dt*1e3:.2f} ms  {mp/dt:.1f} MP/s", {k: round(v, 3) for k, v in st['stage_ms'].items()},
          {k: st[k] for k in ('pairs', 'streamed', 'popped', 'composited', 'reject_radius', 'reject_bracket', 'fp64_evals', 'fp64_pixels', 'ambiguous', 'ring_miss', 'poly_overflow', 'launches', 'cache_appends', 'tie_runs', 'tie_members', 'tie_max_run')}, flush=True)
    if scenes.CONFIGS[cfg]['backward']:
        tgt = torch.from_numpy(scenes.config_target(cfg, cam).astype(np.float32)).cuda()
        for _ in range(2):
            fb = r.render(raw, cam, opt); v, d = r.l1_loss(fb.color, tgt); g = r.backward_render(raw, FrameGrad(d_color=d))
        torch.cuda.synchronize(); t = time.time()
        for _ in range(N):
            fb = r.render(raw, cam, opt); v, d = r.l1_loss(fb.color, tgt); g = r.backward_render(raw, FrameGrad(d_color=d))
        torch.cuda.synchronize(); dt = (time.time() - t) / N
        st = r.stats()
        print(f"cfg{cfg} fwd+bwd {dt*1e3:.2f} ms  {mp/dt:.1f} MP/s loss {float(v):.4f}",
              {k: round(v, 3) for k, v in st['stage_ms'].items()}, 'warpsteps', st['bwd_warp_steps'],
              'lead_records', st['bwd_lead_records'], 'composited', st['composited'], flush=True)
if os.environ.get('DET'):
    # deterministic backward (drk_det.cu) on the last config with a backward
    for cfg in [2]:
        sc = scenes.config_scene(cfg); cam = scenes.config_cameras(cfg)[0]
        raw = torch.from_numpy(sc.f32()).cuda()
        opt = RenderOptions(sh_degree=3)
        tgt = torch.from_numpy(scenes.config_target(cfg, cam).astype(np.float32)).cuda()
        fb = r.render(raw, cam, opt); v, d = r.l1_loss(fb.color, tgt)
        for det in (False, True, True):
            torch.cuda.synchronize(); t = time.time()
            g = r.backward_render(raw, FrameGrad(d_color=d), deterministic=det)
            torch.cuda.synchronize()
            print(f"cfg{cfg} backward deterministic={det}: {1e3 * (time.time() - t):.1f} ms", flush=True)
