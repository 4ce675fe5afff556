"""adapter_bench on config 2 with DRK_ADAPTER_TRACE=1 (phase times of the drop-in calls)."""
import os, subprocess, sys, tempfile
import numpy as np
sys.path.insert(0, '.')
from paper_2412_11752_b200 import scenes
prec = sys.argv[1] if len(sys.argv) > 1 else "fast"
sc = scenes.config_scene(2)
cam = scenes.config_cameras(2)[0]
tgt = scenes.config_target(2, cam)
with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as fh:
    fh.write(np.array([sc.n, sc.k, sc.terms, cam.width, cam.height], np.int32).tobytes())
    fh.write(np.concatenate([[cam.fx, cam.fy, cam.cx, cam.cy], np.asarray(cam.R).ravel(),
                             np.asarray(cam.t).ravel()]).astype(np.float64).tobytes())
    fh.write(sc.f32().tobytes())
    fh.write(np.ascontiguousarray(tgt, np.float64).tobytes())
    path = fh.name
env = dict(os.environ, DRK_ADAPTER_PRECISION=prec, DRK_ADAPTER_TRACE="1")
r = subprocess.run(["oracle/_ref/adapter_bench", path, "1", "2"], capture_output=True, text=True, env=env)
print(prec, r.stdout.strip())
print(r.stderr[-3000:])
