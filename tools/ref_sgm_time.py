"""Reference SGM on the host (measurement tool): oracle/_ref's sgm_disparity on one C2 frame."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle_lib
from paper_2604_07980_b200 import synth as S
ref = oracle_lib.reference()
sc, _ = S.scene_c2(seed=1, noise=2.0)
L, R = S.render_stereo_pair(sc)
out = np.zeros_like(L, dtype=np.int16)
t = time.perf_counter()
st = ref.lib.ref_sgm_disparity(L.ctypes.data, R.ctypes.data, 1920, 1080, 64, 0, 8, 32, out.ctypes.data)
print({"ref_sgm_seconds_per_frame_1thread": round(time.perf_counter() - t, 2), "status": st})
