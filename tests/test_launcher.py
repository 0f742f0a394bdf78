"""bench.py --gpus N without torchrun: the launcher starts N rank processes
with torchrun's environment (CPU test: a stand-in script records what each
rank sees, then the ranks rendezvous over gloo and all_reduce)."""

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

RANK_SCRIPT = r'''
import json, os, sys
import torch
import torch.distributed as dist
out = sys.argv[1]
env = {k: os.environ.get(k) for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE",
                                       "MASTER_ADDR", "MASTER_PORT", "NCCL_DEBUG")}
dist.init_process_group("gloo")
t = torch.tensor([int(env["RANK"]) + 1.0])
dist.all_reduce(t)
env["sum"] = float(t.item())
env["world"] = dist.get_world_size()
dist.destroy_process_group()
open(os.path.join(out, f"rank{env['RANK']}.json"), "w").write(json.dumps(env))
'''


def test_spawn_ranks_environment(tmp_path):
    import bench
    script = tmp_path / "rank.py"
    script.write_text(RANK_SCRIPT)
    rc = bench.spawn_ranks(2, argv=[str(tmp_path)], script=script)
    assert rc == 0
    seen = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(2)]
    for r, e in enumerate(seen):
        assert e["RANK"] == str(r) and e["LOCAL_RANK"] == str(r)
        assert e["WORLD_SIZE"] == "2" and e["MASTER_ADDR"] == "127.0.0.1"
        assert e["world"] == 2 and e["sum"] == 3.0
        assert e["NCCL_DEBUG"]   # the communicator log is on (INFO unless the caller set it)
    assert seen[0]["MASTER_PORT"] == seen[1]["MASTER_PORT"]


def test_spawn_ranks_propagates_failure(tmp_path):
    import bench
    script = tmp_path / "fail.py"
    script.write_text("import os, sys\nsys.exit(3 if os.environ['RANK'] == '1' else 0)\n")
    assert bench.spawn_ranks(2, argv=[], script=script) == 3
