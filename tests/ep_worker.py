"""One expert-parallel rank in its own process (tests/test_ep_processes.py).

Every rank builds the same device-initialised model, holds only its experts, attaches a transport
and runs run_specmoe + forward; the result (tokens, routing trace, ledger, outcomes, logits digest) is
written as JSON.  --world 1 produces the single-GPU answer the ranks must reproduce bit for bit.

Transports: `host` = the C ABI's host transport over a torch.distributed gloo all-gather (CUDA IPC
handles for the fused peer-memory exchange travel through it; the ranks may share one GPU, and no host
fence sits between a rank's device-side signal and its peers' device-side waits); `nccl` = one GPU
per rank, the NCCL unique id broadcast over gloo."""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {
    "c1": dict(spec=dict(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, gate_skew=1.0, seed=1,
                         expert_kind=1),
               B=3, n_draft=4, new=16),
    "e64": dict(spec=dict(num_layers=3, experts=64, top_k=6, hidden=256, ffn=256, vocab=512, expert_kind=1,
                          moe_mask=[0, 1, 1], gate_skew=0.5, seed=4),
                B=5, n_draft=8, new=12),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--port", type=int, default=29611)
    ap.add_argument("--transport", default="host", choices=["host", "nccl"])
    ap.add_argument("--mode", default="p2p", choices=["p2p", "a2a"])
    ap.add_argument("--shape", default="c1", choices=list(SHAPES))
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    os.environ["SMOE_EP_MODE"] = a.mode
    from paper_2604_10152_b200.engine import BF16, Engine, HostTransport, ModelSpec, RunCfg, gloo_allgather
    from paper_2604_10152_b200.prompts import make_prompts

    sh = SHAPES[a.shape]
    spec = ModelSpec(**sh["spec"])
    prompts = make_prompts(8, sh["B"], 8, spec.vocab)
    cfg = RunCfg(gamma=4, n_draft=sh["n_draft"], max_new_tokens=sh["new"], collect_trace=True)
    dev = a.rank if a.transport == "nccl" else 0
    if a.world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{a.port}", rank=a.rank, world_size=a.world)
    e = Engine(spec, weight_type=BF16, max_batch=sh["B"], max_gamma=4, device=dev,
               ep_rank=a.rank if a.world > 1 else 0, ep_world=a.world)
    e.init_device(13)
    e.build_affinity_device()
    if a.world > 1:
        if a.transport == "host":
            e.attach_host(HostTransport(gloo_allgather()))
        else:
            from paper_2604_10152_b200.engine import nccl_unique_id
            obj = [nccl_unique_id() if a.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            e.attach_nccl(obj[0])
    r = e.run_specmoe(cfg, prompts)
    od = e.run_ondemand(cfg, prompts)
    lg, raw, fin = e.forward(prompts[2] + [7, 9])
    out = {"tokens": r.tokens, "trace": [list(t[:3]) + [list(t[3])] for t in r.trace],
           "ledger": [list(x) for x in r.ledger], "outcomes": [list(o[:5]) + [list(o[5])] for o in r.outcomes],
           "ondemand_tokens": od.tokens, "tau": r.metrics["tau_mean"],
           "logits_sha": hashlib.sha256(lg.tobytes()).hexdigest(), "raw": raw.tolist(), "fin": fin.tolist()}
    with open(a.out, "w") as f:
        json.dump(out, f)
    e.close()
    if a.world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
