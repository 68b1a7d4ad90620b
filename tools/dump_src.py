"""Write the NVRTC translation units of the bench modules next to the repo
root under the names NVRTC compiled them with, so `ncu --page source`
can resolve -lineinfo lines (cprrtc-*.cu are git-ignored)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import fixtures as fx
from paper_2505_06791_b200 import _lib

MODS = [("arm7", 16, 0, 1, 0), ("arm7", 16, 0, 0, 1)]
for name, G, kind, orient, parity in MODS:
    src = _lib.device_source(fx.robot(name).packed, G, kind, orient, parity)
    fn = os.path.join(ROOT, f"cprrtc-{'parity' if parity else 'plan'}-g{G}-k{kind}-o{orient}.cu")
    with open(fn, "w") as fh:
        fh.write(src)
    print(fn, len(src))
