import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from paper_1809_07986_b200 import tsgm
from paper_1809_07986_b200.scene import SceneConfig, render
S, F, H, W = 64, 30, 375, 1242
calib = tsgm.StereoCalib(720.0, 621.0, 187.5, 0.54, W, H, 128)
eng = tsgm.Engine(tsgm.EngineConfig(calib, tsgm.SgmParams(10, 120, 8, 0, 128),
                                    tsgm.FilterConfig(range_use_stddev=True, range_stddev_gain=3.0), max_slots=S, keep_volumes=False))
hl = torch.empty((S, F, H, W), dtype=torch.uint8).pin_memory(); hr = torch.empty_like(hl).pin_memory()
mot = []
for s in range(S):
    L, R, P, _ = render(SceneConfig.baseline_config(2, seed=s, n_movers=s % 5, frames=F), out_left=hl[s].numpy(), out_right=hr[s].numpy())
    mot.append([(np.eye(3), np.zeros(3)) if k == 0 else tsgm.relative_motion(P[k - 1], P[k]) for k in range(F)])
dl, dr = hl.cuda(), hr.cuda()
HL, HR = hl.numpy(), hr.numpy()
outs = {k: torch.empty((S, H, W), dtype=dt).pin_memory().numpy() for k, dt in
        (("export_d", torch.int32), ("export_valid", torch.uint8), ("state_p", torch.float64), ("mask", torch.uint8))}
slots = list(range(S))
m12 = np.zeros((F, S, 12))
for k in range(F):
    for i in range(S):
        m12[k, i, :9] = mot[i][k][0].ravel(); m12[k, i, 9:] = mot[i][k][1]
def run(host, fetch):
    for s in slots: eng.reset(s)
    for k in range(F):
        if host:
            eng.step(slots, [HL[i, k] for i in slots], [HR[i, k] for i in slots], [mot[i][k] for i in slots])
        else:
            eng.step_device(slots, [dl[i, k].data_ptr() for i in slots], [dr[i, k].data_ptr() for i in slots], m12[k])
        if fetch:
            for key, arr in outs.items():
                eng.fetch_batch(slots, key, [arr[i] for i in slots])
    eng.sync()
for name, host, fetch in (("device", False, False), ("host_in", True, False), ("device_fetch", False, True), ("host_fetch", True, True)):
    run(host, fetch)
    t = time.perf_counter()
    for _ in range(2): run(host, fetch)
    dt = (time.perf_counter() - t) / 2
    print(name, round(S * F / dt, 1), "frames/s", round(dt * 1e3, 1), "ms/step", flush=True)
