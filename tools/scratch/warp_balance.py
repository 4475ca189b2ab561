import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2511_21669_b200 import Simulator
s = Simulator(0)
n, p = s.prepare_sweep("configs/c5_sweep_65536.yaml")
s.launch(); s.sync()
ev = s.summaries()["events_processed"].astype(np.float64)
w = ev[: len(ev) // 32 * 32].reshape(-1, 32)
mx, mean = w.max(1), w.mean(1)
print("replica events: min %d mean %.0f max %d" % (ev.min(), ev.mean(), ev.max()))
print("lane efficiency within warps (sum/ (32*max)): %.3f" % (w.sum() / (32 * mx).sum()))
print("warp max-lane events quantiles:", np.percentile(mx, [10, 50, 90, 99, 100]).astype(int))
# per-SM (one wave): warps are dealt to SMs by block id; 2 warps per block
np.save("gpurun_out/c5_events.npy", ev)
