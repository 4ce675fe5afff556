#!/bin/bash
# round 2 session 20: copy-out path in a fresh process (timing on / off)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
O=gpurun_out/r2s20
cat > /tmp/hang_probe.py <<'PY'
import faulthandler, sys, os
faulthandler.dump_traceback_later(40, exit=True)
sys.argv = ['x', '1']
if os.environ.get('TIMING') == '1':
    import paper_2412_11752_b200.api as api
    orig = api.Rasterizer.__init__
    def init(self, *a, **k):
        orig(self, *a, **k); self.set_timing(True)
    api.Rasterizer.__init__ = init
exec(open('scripts/e2e_probe.py').read())
PY
DRK_HOST_OUT=copy TIMING=1 DRK_HOST_TRACE=1 timeout 60 python /tmp/hang_probe.py > $O.t1.log 2>&1; echo "rc=$?" >> $O.t1.log
DRK_HOST_OUT=copy TIMING=0 DRK_HOST_TRACE=1 timeout 60 python /tmp/hang_probe.py > $O.t0.log 2>&1; echo "rc=$?" >> $O.t0.log
