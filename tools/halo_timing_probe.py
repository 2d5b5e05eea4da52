"""Device time of one band exchange (pack kernel, NCCL all-gather, unpack
kernel) with one rank, CUDA events on the current stream (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29535", RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_1810_05628_b200 import sharding, _lib  # noqa: E402

n, ov = 512, 48
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
g = torch.randn(n, n, dtype=torch.complex64, device="cuda")
v = torch.zeros(4, dtype=torch.float64, device="cuda")
ex = sharding.HaloExchange(n, ov, torch.complex64, "cuda")
lib = _lib.lib()
for _ in range(50):
    ex(g, v)
torch.cuda.synchronize()
for name, fn in [("pack", lambda: lib.ptg_halo_pack(0, g.data_ptr(), n, ov, v.data_ptr(), ex.buf.data_ptr(), stream.cuda_stream)),
                 ("all_gather", lambda: dist.all_gather_into_tensor(ex.all, ex.buf)),
                 ("unpack", lambda: lib.ptg_halo_unpack(0, g.data_ptr(), n, ov, ex.all.data_ptr(), 0, 1, v.data_ptr(), stream.cuda_stream)),
                 ("full exchange", lambda: ex(g, v))]:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(200):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us")
dist.destroy_process_group()
