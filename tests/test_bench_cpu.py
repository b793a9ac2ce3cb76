"""bench.py host logic without a GPU: the --gpus N self-launch (torchrun
re-exec), the refusal when the node has fewer GPUs than asked, and the
JSON keys the driver compares between the two arms."""
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_torchrun_cmd_reexecs_bench_with_same_args():
    argv = ["--gpus", "4", "--steps", "7", "--warmup", "3"]
    cmd = bench.torchrun_cmd(argv, 4, 29512)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nnodes=1" in cmd and "--nproc-per-node=4" in cmd
    i = cmd.index("--master-addr")
    assert cmd[i + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29512"
    script = os.path.abspath(os.path.join(ROOT, "bench.py"))
    assert cmd[cmd.index(script) + 1:] == argv


def test_gpus_more_than_present_fails_loudly():
    # this container has no GPU: --gpus 2 must refuse, not print a 1-GPU line labelled 2 GPUs
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode != 0
    assert "needs 2 GPUs" in p.stderr
    assert '"value"' not in p.stdout


def test_config_has_no_arm_specific_keys():
    # the driver compares `config` between our arm and the reference arm
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'config["l2_bytes"]' not in src
