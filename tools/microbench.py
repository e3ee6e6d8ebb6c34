"""Run the pipe microbenchmarks of libvqb200.so and print one JSON line."""
import ctypes, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0910_4711_b200 import _lib
L = _lib.lib()
out = {}
import os as _os
sel = [int(v) for v in _os.environ.get("MB_ONLY", "").split(",") if v]
for which, name in [(0, "ffma"), (1, "ffma2"), (2, "ffma_top2_mix"), (3, "dadd"), (4, "ffma_3reg"), (5, "dist_const_evals"), (6, "ffma2_plus_ffma"), (7, "fmnmx"), (8, "fmnmx_2reg"), (9, "vimnmx_2reg"), (10, "fmnmx_plus_vimnmx"), (11, "smem_red_random"), (12, "smem_atom_return_random"), (13, "xread_row_per_lane_Bps"), (14, "xread_coalesced_Bps"), (15, "l2_red64_k1024x17"), (16, "l2_red64_k4096x17"), (17, "fmnmx3_3reg"), (18, "fmnmx3_plus_fold")]:
    if sel and which not in sel:
        continue
    for bps in (2, 4):
        ops = ctypes.c_double(); sec = ctypes.c_double()
        _lib.check(L.vqb_pipe_microbench(which, bps, 4000, ctypes.byref(ops), ctypes.byref(sec)))
        out[f"{name}_bps{bps}_Gops"] = round(ops.value / 1e9, 1)
        out[f"{name}_bps{bps}_ms"] = round(sec.value * 1e3, 3)
print(json.dumps(out))
