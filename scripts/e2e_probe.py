"""e2e (drk_forward_host) timing of config 1 under the host-buffer modes
(DRK_HOST_OUT=copy|map-default, DRK_HOST_IN=map) and a digest of the outputs."""
import hashlib, os, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
from paper_2412_11752_b200.api import Rasterizer, RenderOptions

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
r = Rasterizer(0)
sc = scenes.config_scene(cfg)
cam = scenes.config_cameras(cfg)[0]
opt = RenderOptions(sh_degree=scenes.CONFIGS[cfg]['sh_degree'])
host_raw = torch.from_numpy(sc.f32()).pin_memory()
outs = {"color": torch.empty(cam.height, cam.width, 3, pin_memory=True),
        "depth": torch.empty(cam.height, cam.width, pin_memory=True),
        "normal": torch.empty(cam.height, cam.width, 3, pin_memory=True),
        "alpha": torch.empty(cam.height, cam.width, pin_memory=True)}
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
stream = torch.cuda.current_stream()
for _ in range(3):
    r.render_host_ptrs(host_raw, outs, cam, opt)
ms = []
for _ in range(10):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    r.render_host_ptrs(host_raw, outs, cam, opt)
    b.record(stream)
    b.synchronize()
    ms.append(a.elapsed_time(b))
h = hashlib.sha1()
for k in ("color", "depth", "normal", "alpha"):
    h.update(outs[k].numpy().tobytes())
# device path for reference
fb = r.render(host_raw.cuda(), cam, opt)
same = all(torch.equal(getattr(fb, k).cpu().reshape(outs[k].shape), outs[k]) for k in ("color", "depth", "normal", "alpha"))
px = cam.width * cam.height
print(f"mode out={os.environ.get('DRK_HOST_OUT', 'map')} in={os.environ.get('DRK_HOST_IN', 'copy')} cfg{cfg}: "
      f"median {np.median(ms):.3f} ms  min {min(ms):.3f}  {px / np.median(ms) / 1e3:.1f} MP/s  digest {h.hexdigest()[:16]}  equal_to_device {same}",
      flush=True)
