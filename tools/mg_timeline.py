"""Multi-GPU timeline (development tool): per-exchange active explorers per rank."""
import os, sys, time, json
sys.path.insert(0, ".")
import torch, torch.distributed as dist
import paper_2012_09511_b200 as pbb
from paper_2012_09511_b200 import multi

local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()
name, ub, bound = sys.argv[1], int(sys.argv[2]), sys.argv[3]
low = float(sys.argv[4]) if len(sys.argv) > 4 else 0.25
pinned = len(sys.argv) > 5 and sys.argv[5] == "pinned"
X = int(sys.argv[6]) if len(sys.argv) > 6 else None
quiet = len(sys.argv) > 7
pool = pbb.GpuPool(pbb.taillard_named(name), pbb.PoolConfig(device=local, pinned=pinned, split_mode=int(os.environ.get("SPLIT_MODE", "0"))), bound=bound)
multi.solve_distributed(pool, ub, device=dev, low_fraction=low, export_max=X)  # warm
log = []
orig = pool.run_round
t0 = [0.0]
def rr():
    a = orig()
    log.append((round(time.time() - t0[0], 4), a))
    return a
pool.run_round = rr
dist.barrier(); torch.cuda.synchronize(); t0[0] = time.time()
r = multi.solve_distributed(pool, ub, device=dev, low_fraction=low, export_max=X)
torch.cuda.synchronize(); dt = time.time() - t0[0]
allg = [None] * world
dist.all_gather_object(allg, log)
if rank == 0:
    print(json.dumps({"world": world, "low": low, "s": round(dt, 4), "unique": r.unique, "remote": r.remote_intervals, "rounds": r.rounds}))
    for i in (range(max(len(x) for x in allg)) if not quiet else []):
        print(i, " ".join(f"{x[i][0]:.3f}:{x[i][1]:5d}" if i < len(x) else "-" for x in allg))
dist.destroy_process_group()
