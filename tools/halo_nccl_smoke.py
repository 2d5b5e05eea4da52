import os, sys
sys.path.insert(0, ".")
import torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_1810_05628_b200 import sharding
n, ov = 512, 48
g = torch.randn(n, n, dtype=torch.complex64, device="cuda")
v = torch.tensor([3.5, 0, 0, 0], dtype=torch.float64, device="cuda")
g0 = g.clone()
ex = sharding.HaloExchange(n, ov, torch.complex64, "cuda")
ex(g, v)
torch.cuda.synchronize()
print("world1 nccl halo ok:", torch.equal(g, g0), float(v[0]))
dist.destroy_process_group()
