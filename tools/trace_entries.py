"""Per-ring-entry timeline of CTA 0 for one steady layer launch (library
built with -DSPDNN_TRACE; diagnostics, never a bench number).

    SPDNN_NVCC_DEFINES=-DSPDNN_TRACE python tools/trace_entries.py c2 --layer 200 [--ablate]

Replays the layer like tools/layer_ablate.py, then prints, per entry k, the
times (us, relative to entry 0's grant) of: grant (rows free), gathers
issued, units of k-nbuf done, publisher done, header posted, and the start /
loop end / unit end of consumer warp 0 and of the last consumer warp, plus
the per-stage averages over the steady entries.
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv = [a for a in sys.argv]
# reuse the replay of layer_ablate (it runs the layer 20 times)
import runpy  # noqa: E402

runpy.run_path(os.path.join(ROOT, "tools", "layer_ablate.py"), run_name="__main__")

from paper_2007_14152_b200 import _native  # noqa: E402

lib = _native.lib()
buf = (ctypes.c_int64 * (96 * 12))()
_native.check(lib.spdnn_trace_read(buf, 96 * 12), "spdnn_trace_read")
t = np.array(list(buf), dtype=np.float64).reshape(96, 12)
ghz = 1.965e3  # clocks per us
n = int((t[:, 0] > 0).sum())
if n == 0:
    print("no trace (build with -DSPDNN_TRACE)")
    sys.exit(0)
t0 = t[0, 0]
rel = np.where(t > 0, (t - t0) / ghz, np.nan)
names = ["grant", "gathers", "empty", "free", "posted", "w0 start", "w0 loop", "w0 done",
         "wL start", "wL loop", "wL done", "pub empty"]
print("k     " + " ".join(f"{x:>9s}" for x in names))
for k in range(min(n, 40)):
    print(f"{k:3d} " + " ".join(f"{v:9.2f}" for v in rel[k]))
ks = np.arange(6, min(n, 90))
d = lambda a, b: np.nanmean(rel[ks, a] - rel[ks, b])
nb = 2
print("steady entries", ks[0], "..", ks[-1])
print(f"  grant -> gathers issued     {d(1, 0):6.2f} us")
print(f"  grant -> header posted      {d(4, 0):6.2f} us")
print(f"  header -> w0 start          {d(5, 4):6.2f} us")
print(f"  w0 start -> w0 loop end     {d(6, 5):6.2f} us   (last warp {d(9, 8):6.2f})")
print(f"  w0 loop end -> unit end     {d(7, 6):6.2f} us   (last warp {d(10, 9):6.2f})")
print(f"  w0 start vs last start      {d(8, 5):6.2f} us")
print(f"  entry period (grant k+1 - grant k) {np.nanmean(np.diff(rel[ks, 0])):6.2f} us")
# slot turnaround: entry k's last unit done -> entry k+nb granted
turn = rel[ks[:-nb] + nb, 0] - np.fmax(rel[ks[:-nb], 7], rel[ks[:-nb], 10])
print(f"  units of k done -> grant k+{nb} {np.nanmean(turn):6.2f} us (rows are granted at loop end)")
