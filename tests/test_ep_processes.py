"""Expert parallelism with one OS process per rank, real concurrency.

The loopback tests in test_engine_gpu.py drive G virtual ranks from G threads of one process and add a
host fence after every device-side signal, so the flag protocol of the fused peer-memory exchange
(k_ep_signal's st.release.sys / k_ep_wait's polls) never races anything there.  Here every rank is its
own process with its own CUDA context; the fused exchange's buffers are opened from CUDA IPC handles
that travel over a gloo all-gather (the C ABI's host transport), and no host synchronisation sits
between a rank's signal and its peers' waits.  The ranks share the box's GPU(s): with one GPU the two
contexts time-slice, so every wait genuinely spins until the other process's kernels run.

Bar: token streams, routing trace, ledger, outcomes and forward() logits of every rank equal the
single-GPU run bit for bit, for both exchange paths (p2p peer stores, a2a collectives over the host
transport), on the C1-like and the fine-grained E64/K6 shapes.  With >= 2 GPUs the NCCL transport is
exercised the same way."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
WORKER = os.path.join(HERE, "ep_worker.py")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(tmp_path, world, shape, mode="p2p", transport="host", timeout=400):
    port = _port()
    procs, outs = [], []
    for r in range(world):
        out = str(tmp_path / f"{shape}_{mode}_{transport}_{world}_{r}.json")
        outs.append(out)
        procs.append(subprocess.Popen(
            [sys.executable, WORKER, "--rank", str(r), "--world", str(world), "--port", str(port), "--shape", shape,
             "--mode", mode, "--transport", transport, "--out", out],
            stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=timeout)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [json.load(open(o)) for o in outs]


_SINGLE = {}


def _single(tmp_path, shape):
    if shape not in _SINGLE:
        _SINGLE[shape] = _launch(tmp_path, 1, shape)[0]
    return _SINGLE[shape]


@pytest.mark.parametrize("shape", ["c1", "e64"])
@pytest.mark.parametrize("mode", ["p2p", "a2a"])
def test_ep_two_processes_bitexact(tmp_path, shape, mode):
    want = _single(tmp_path, shape)
    assert want["tokens"] == want["ondemand_tokens"]
    for got in _launch(tmp_path, 2, shape, mode=mode):
        for k in ("tokens", "trace", "ledger", "outcomes", "ondemand_tokens", "logits_sha", "raw", "fin"):
            assert got[k] == want[k], (shape, mode, k)


def _gpus():
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        return sum(1 for l in out.splitlines() if l.startswith("GPU "))
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="NCCL transport needs >= 2 GPUs (NCCL refuses two ranks on one device)")
@pytest.mark.parametrize("mode", ["p2p", "a2a"])
def test_ep_nccl_two_gpus_bitexact(tmp_path, mode):
    want = _single(tmp_path, "c1")
    for got in _launch(tmp_path, 2, "c1", mode=mode, transport="nccl"):
        for k in ("tokens", "trace", "ledger", "outcomes", "logits_sha"):
            assert got[k] == want[k], (mode, k)
