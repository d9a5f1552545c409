"""Time parm_peer_barrier variants (library builds) at P = WORLD_SIZE, graph of back-to-back barriers.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/probes/barrier_probe.py [lib.so ...]
"""
import ctypes
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2407_00599_b200 import _lib  # noqa: E402
from paper_2407_00599_b200.config import ParallelLayout  # noqa: E402
from paper_2407_00599_b200.peer_calibrate import _time  # noqa: E402
from paper_2407_00599_b200.world import PeerWorld  # noqa: E402


def load_any(path):
    lib = ctypes.CDLL(path)
    for name, (res, args) in _lib.SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.restype, fn.argtypes = res, args
    return lib


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P = dist.get_world_size()
    world = PeerWorld(ParallelLayout(P // 2 if P > 1 else 1, 1, 2 if P > 1 else 1, P) if P == 2 else
                      ParallelLayout(2, P // 2, 2, P) if P == 4 else ParallelLayout(1, 1, 1, 1), dev)
    base = _lib.load()
    for path in [None] + sys.argv[1:]:
        _lib._lib = base if path is None else load_any(path)
        t = [_time(world.peer_barrier, dev, reps=9, inner=16) for _ in range(3)]
        if dist.get_rank() == 0:
            print(f"{Path(path).name if path else 'in-tree':>12s}  barrier {min(t) * 1e6:6.2f} us  (runs {[round(x * 1e6, 2) for x in t]})",
                  flush=True)
    dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
