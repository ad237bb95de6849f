"""Multi-GPU launch plumbing on the CPU (no torch.distributed anywhere):

* distributed.launch() starts one process per rank with RANK / LOCAL_RANK /
  WORLD_SIZE and one shared NCCL id (LGP_NCCL_ID),
* the rendezvous-file id exchange used under torchrun (rank 0 publishes, the
  others read the same 128 bytes),
* bench.py --gpus N refuses to fake N ranks: without enough GPUs it fails
  loudly, and under a launcher whose WORLD_SIZE disagrees with --gpus too.
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, os, sys
sys.path.insert(0, {root!r})
from paper_2605_17898_b200 import distributed
rank, world, local = distributed.env_rank_world()
ident, owned = distributed.exchange_id(rank, world)
with open(os.path.join({out!r}, f"rank{{rank}}.json"), "w") as f:
    json.dump(dict(rank=rank, world=world, local=local, id=ident.hex(),
                   env_id=os.environ.get("LGP_NCCL_ID", "")), f)
print(f"rank {{rank}} stdout")
"""


def test_launch_ranks_share_one_id(tmp_path):
    from paper_2605_17898_b200 import distributed

    out = tmp_path / "res"
    out.mkdir()
    stdout = tmp_path / "stdout.txt"
    with open(stdout, "w") as f:
        code = distributed.launch([sys.executable, "-c", PROBE.format(root=ROOT, out=str(out))],
                                  3, stdout_rank0=f)
    assert code == 0
    res = [json.load(open(out / f"rank{r}.json")) for r in range(3)]
    assert [r["rank"] for r in res] == [0, 1, 2]
    assert all(r["world"] == 3 and r["local"] == r["rank"] for r in res)
    assert len({r["id"] for r in res}) == 1 and len(res[0]["id"]) == 256
    assert res[0]["id"] == res[0]["env_id"]
    # only rank 0's stdout is forwarded (bench.py prints one JSON line)
    assert open(stdout).read().split() == ["rank", "0", "stdout"]


def test_rendezvous_file_exchange(tmp_path):
    out = tmp_path / "res"
    out.mkdir()
    env = {k: v for k, v in os.environ.items() if k != "LGP_NCCL_ID"}
    env["LGP_RDZV_FILE"] = str(tmp_path / "nccl-id")
    procs = []
    for r in (2, 1, 0):  # readers start first and wait for rank 0
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="3")
        procs.append(subprocess.Popen([sys.executable, "-c", PROBE.format(root=ROOT, out=str(out))],
                                      env=e, stdout=subprocess.DEVNULL))
    assert all(p.wait(timeout=120) == 0 for p in procs)
    res = [json.load(open(out / f"rank{r}.json")) for r in range(3)]
    assert len({r["id"] for r in res}) == 1 and len(res[0]["id"]) == 256
    assert all(r["env_id"] == "" for r in res)


def _bench(args, env=None):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                          capture_output=True, text=True, timeout=300, cwd=ROOT,
                          env=env)


def test_bench_gpus_without_gpus_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")}
    r = _bench(["--gpus", "2", "--steps", "3"], env=env)
    assert r.returncode == 2 and "visible GPUs" in r.stderr
    assert r.stdout.strip() == ""


def test_bench_gpus_must_match_launcher_world():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = _bench(["--gpus", "4", "--steps", "3"], env=env)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_bench_reference_arm_n_gpus_label():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")}
    r = _bench(["--impl", "reference", "--gpus", "4", "--config", "cfg1", "--steps", "1",
                "--warmup", "0"], env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["n_gpus"] == 4


def test_product_path_imports_no_torch():
    code = ("import sys; sys.path.insert(0, %r); import paper_2605_17898_b200, "
            "paper_2605_17898_b200.distributed, paper_2605_17898_b200.server; "
            "print('torch' in sys.modules)" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "False"
