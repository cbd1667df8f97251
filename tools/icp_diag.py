"""Diagnostic: ICP iteration-by-iteration GPU vs oracle from identical maps."""
import sys, ctypes as C
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import numpy as np
import vf_py
from helpers import frames
from paper_1410_0925_b200 import make_pipeline, settings_from_config
from paper_1410_0925_b200.scene import CONFIGS
olib = vf_py.oracle_lib()
base = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
fr = frames(olib, base, 3)
o0 = vf_py.Volume(olib, base, tracking=False)
for pose, depth, _ in fr[:2]:
    o0.process(depth, None, pose)
pts, nrm = o0.maps(); rp = o0.pose()
for levels, iters in [(1, 1), (1, 2), (1, 3), (1, 5), (2, 3), (5, 20)]:
    cfg = base.with_(levels=levels, max_iterations=iters, rotation_only_levels=min(2, levels - 1))
    o = vf_py.Volume(olib, cfg, tracking=False)
    olib.lib.vfo_set_maps(o.h, pts.ctypes.data_as(C.c_void_p), nrm.ctypes.data_as(C.c_void_p), rp.ctypes.data_as(C.c_void_p))
    s, c = settings_from_config(cfg)
    p = make_pipeline(s, c)
    p.set_maps(pts, nrm, rp)
    depth = fr[2][1]
    res = p.icp_track(depth)
    out = np.zeros(12); it, cost, valid = C.c_int(), C.c_double(), C.c_int()
    ok = olib.lib.vfo_stage_icp(o.h, depth.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p), C.byref(it), C.byref(cost), C.byref(valid))
    tg = p.icp_trace(); to = np.zeros((512, 32)); n = olib.lib.vfo_icp_trace(o.h, to.ctypes.data_as(C.c_void_p), 512)
    print(f"levels={levels} iters={iters} ok={res['ok']},{ok} it={res['iterations']},{it.value} dpose={np.abs(res['pose']-out).max():.3e} rows={len(tg)},{n}")
    for k in range(min(len(tg), n)):
        rg, ro = tg[k], to[k]
        dh = np.abs(rg[2:23]-ro[2:23]).max()/np.abs(ro[2:23]).max()
        dg = np.abs(rg[23:29]-ro[23:29]).max()/max(np.abs(ro[23:29]).max(),1e-300)
        print(f"   row{k} L{int(ro[0])} i{int(ro[1])} cnt={int(rg[30])},{int(ro[30])} dH={dh:.2e} dg={dg:.2e} dcost={abs(rg[29]-ro[29])/ro[29]:.2e} |g|={np.abs(ro[23:29]).max():.3e}")
    p.close(); o.close()
