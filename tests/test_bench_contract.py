"""bench.py's reference arm on CPU (config 2, seconds): the JSON line carries the contract's keys
(the GPU arm's line is checked on the GPU box by running bench.py itself)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "2",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert "workload" in line["config"]


def test_gpus_flag_fails_loudly_without_enough_gpus():
    """`bench.py --gpus 2` outside torchrun self-launches one rank per GPU -- and refuses (exit 2, a
    message on stderr) when fewer GPUs are visible, instead of silently running one rank."""
    import torch
    if torch.cuda.device_count() >= 2:
        import pytest
        pytest.skip("two GPUs visible: the self-launch would run")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 2 and "visible GPUs" in out.stderr, (out.returncode, out.stderr[-500:])
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                         text=True, timeout=300, env={**os.environ, "WORLD_SIZE": "1"})
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stderr


def test_ipm_watchdog_emits_and_exits():
    """The N > 1 IPM leg's watchdog (bench.start_watchdog): when the leg outlives its timeout the line
    is still emitted and the process ends with status 0; a cancelled watchdog never fires."""
    import threading
    sys.path.insert(0, ROOT)
    import bench
    fired, exited = [], threading.Event()
    t = bench.start_watchdog(0.05, lambda: fired.append("line"), exit_fn=lambda code: (fired.append(code), exited.set()))
    assert exited.wait(5.0)
    assert fired == ["line", 0]
    calls = []
    t2 = bench.start_watchdog(0.2, lambda: calls.append(1), exit_fn=lambda code: calls.append(code))
    t2.cancel()
    t2.join(1.0)
    assert calls == []
    t.join(1.0)
