"""Time the band path's block-sweep kernel under its development switches
(bamg_band_sweep_probe): which part of a block step costs what."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1402_4005_b200 import _lib

L = _lib.lib()
c = _lib.ctx()
names = {0: "full", 1: "no global store", 2: "no DSMEM gather", 4: "no cluster barrier", 8: "no prefetch",
         6: "no gather+barrier", 15: "nothing but compute"}
for S, nb, p in [(128, 128, 1), (128, 128, 28), (128, 128, 8)]:
    for dev in (0, 1, 2, 4, 8, 6, 15):
        ms = C.c_double()
        _lib.check(L.bamg_band_sweep_probe(c, S, nb, p, 20, dev, C.byref(ms)), "probe")
        print(f"S={S} nb={nb} p={p:2d} {names[dev]:22s} {ms.value * 1e3:8.1f} us/sweep  {ms.value * 1e3 / nb:6.2f} us/step",
              flush=True)
