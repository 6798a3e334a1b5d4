"""cProfile of the sharded PAGANI driver with a one-rank NCCL communicator: where does the per-iteration plumbing go?"""
import cProfile, os, pstats, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native, sharded

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
comm = sharded.Comm(device=0)
f1 = pb.get_integrand("f1", 8)
cfg = pb.PaganiConfig(rel_tol=1e-6, region_cap=1 << 22)
for _ in range(3):
    sharded.pagani_refine_sharded(f1, cfg, comm, force_collectives=True)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    sharded.pagani_refine_sharded(f1, cfg, comm, force_collectives=True)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
dist.destroy_process_group()
