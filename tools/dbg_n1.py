import ctypes, os, sys, numpy as np
import blocktri_oracle as O
from paper_1108_4181_b200 import BlockTriMatrix, configs, plan_build, plan_solve, _native
from paper_1108_4181_b200.dichotomy import plan_build_arrays
np.set_printoptions(precision=4, suppress=True, linewidth=150)

def rrows(p):
    lib = _native.load(); need = ctypes.c_int64(0)
    lib.btd_plan_export(p.handle, None, ctypes.byref(need), None)
    img = np.empty(need.value, np.uint8)
    lib.btd_plan_export(p.handle, ctypes.c_void_p(img.ctypes.data), ctypes.byref(need), None)
    h = img[:104].view(np.int64)
    return img[104 + h[10]:104 + h[10] + h[11]].view(np.float64)

d, lo, up, f = configs.dominant_numpy(1, 2, 3, seed=5)
C = d[0]
print("inv00", np.linalg.inv(C)[0, 0])
for trial in range(3):
    p = plan_build(BlockTriMatrix(d, lo, up), 1)
    print("n=1 R00", rrows(p)[0])
import torch
p = plan_build_arrays(torch.from_numpy(d).cuda(), torch.from_numpy(lo).cuda(), torch.from_numpy(up).cuda(), 1)
print("n=1 device-matrix R00", rrows(p)[0])
d2 = np.stack([C, np.eye(2)]); z = np.zeros((1, 2, 2))
p = plan_build(BlockTriMatrix(d2, z, z), 1)
print("n=2 R00", rrows(p)[0])
os.environ["BTD_FUSED_TREE"] = "0"
p = plan_build(BlockTriMatrix(d, lo, up), 1)
print("n=1 nofused R00", rrows(p)[0])
for seed in range(8):
    dd, ll, uu, ff = configs.dominant_numpy(1, 2, 1, seed=seed)
    p = plan_build(BlockTriMatrix(dd, ll, uu), 1)
    print("seed", seed, "R", rrows(p)[:2], rrows(p)[8:10], "inv", np.linalg.inv(dd[0]).ravel())
