import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import torch.distributed as dist
from paper_0912_1379_b200 import _native, lct2d as L2
buf = ctypes.create_string_buffer(512); ver = ctypes.c_int()
print("info before", _native.lib().xft_nccl_info(buf, 512, ctypes.byref(ver)), buf.value, ver.value)
store = dist.FileStore("/tmp/ncclstore", 1)
dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
print("info after", _native.lib().xft_nccl_info(buf, 512, ctypes.byref(ver)), buf.value, ver.value)
n = 2048
rng = np.random.default_rng(17)
f = torch.from_numpy((rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(np.complex64)).cuda()
ref = L2.lct2d(f, (1.0, 0.25, 0.0, 1.0), (0.5, 1.5, -0.5, 0.5))
for tr in ("nccl", "capi"):
    got = L2.lct2d_sharded(f, (1.0, 0.25, 0.0, 1.0), (0.5, 1.5, -0.5, 0.5), transport=tr)
    torch.cuda.synchronize()
    print(tr, float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref)))
pg = dist.group.WORLD
print("comm ptr", hex(pg._get_backend(f.device)._comm_ptr()))
dist.destroy_process_group()
