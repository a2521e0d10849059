"""Python host mirror of the B200 engine's C ABI (include/specmoe_b200.h).

The hot path is the sm_100a CUDA library ``lib/libspecmoe_b200.so``; this module only marshals
arguments.  It mirrors the reference's API names (``build_model`` / ``forward`` /
``run_specmoe`` / ``run_ondemand``, /root/reference/proj/core/include/specmoe) so parity tests read
like the reference's own examples.  There is no CPU fallback: if the library or a GPU is missing,
every call raises ``EngineError``.
"""
from __future__ import annotations

import ctypes as C
import os
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SMOE_LIB") or os.path.join(HERE, "lib", "libspecmoe_b200.so")  # override: A/B builds

F32, BF16 = 0, 1
TANH2, SWIGLU3 = 0, 1
GEMM_AUTO, GEMM_SIMT, GEMM_TCGEN05 = 0, 1, 2
POLICIES = {"random": 0, "hot_global": 1, "hot_temporal": 2}
PHASES = {0: "speculation", 1: "verification", 2: "baseline-step"}

# every entry point declared in include/specmoe_b200.h
EXPORTS = ["smoe_last_error", "smoe_engine_create", "smoe_engine_destroy", "smoe_engine_info", "smoe_engine_stream",
           "smoe_init_weights_exact", "smoe_init_weights_device", "smoe_upload_tensor", "smoe_set_affinity",
           "smoe_build_affinity_device", "smoe_get_affinity", "smoe_forward", "smoe_run_specmoe", "smoe_run_ondemand",
           "smoe_run_overlap", "smoe_run_caching",
           "smoe_free_result", "smoe_spec_begin", "smoe_spec_step", "smoe_spec_end", "smoe_counters", "smoe_bench_expert_gemm",
           "smoe_profile_reset", "smoe_profile_stop", "smoe_profile_read", "smoe_counter", "smoe_ep_nccl_unique_id", "smoe_ep_attach_nccl",
           "smoe_ep_loopback_create", "smoe_ep_loopback_destroy", "smoe_ep_attach_loopback", "smoe_ep_attach_host",
           "smoe_make_prompts"]


class EngineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class EngineConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("experts", C.c_int), ("top_k", C.c_int), ("hidden", C.c_int),
                ("ffn", C.c_int), ("vocab", C.c_int), ("gate_skew", C.c_double), ("seed", C.c_uint64),
                ("moe_mask", C.POINTER(C.c_uint8)), ("expert_kind", C.c_int), ("weight_type", C.c_int),
                ("max_batch", C.c_int), ("max_gamma", C.c_int), ("gemm_backend", C.c_int), ("device", C.c_int),
                ("offload", C.c_int), ("hbm_expert_slots", C.c_int), ("ep_rank", C.c_int), ("ep_world", C.c_int),
                ("attn_heads", C.c_int), ("kv_heads", C.c_int), ("head_dim", C.c_int), ("rope_theta", C.c_double),
                ("max_seq_len", C.c_int)]


class RunConfig(C.Structure):
    _fields_ = [("gamma", C.c_int), ("n_draft", C.c_int), ("max_new_tokens", C.c_int), ("use_affinity", C.c_int),
                ("warmup_steps", C.c_int), ("policy", C.c_int), ("collect_trace", C.c_int), ("run_seed", C.c_uint64),
                ("device_capacity_bytes", C.c_uint64), ("bytes_per_expert", C.c_uint64),
                ("host_bandwidth", C.c_double), ("ssd_bandwidth", C.c_double), ("compute_rate", C.c_double),
                ("compute_cost_per_expert", C.c_double), ("mode", C.c_int), ("temperature", C.c_double)]


class LedgerEntry(C.Structure):
    _fields_ = [("phase", C.c_int), ("step", C.c_int), ("layer", C.c_int), ("expert", C.c_int), ("bytes", C.c_uint64)]


LEDGER_DTYPE = np.dtype(LedgerEntry)


class Outcome(C.Structure):
    _fields_ = [("seq", C.c_int), ("phase", C.c_int), ("accepted", C.c_int), ("correction", C.c_int),
                ("tokens_generated", C.c_int)]


class RunResultC(C.Structure):
    _fields_ = [("B", C.c_int), ("max_new", C.c_int), ("moe_layers", C.c_int), ("experts", C.c_int),
                ("top_k", C.c_int), ("gamma", C.c_int),
                ("tokens", C.POINTER(C.c_int)), ("n_tokens", C.POINTER(C.c_int)),
                ("n_ledger", C.c_int), ("ledger", C.POINTER(LedgerEntry)),
                ("n_outcomes", C.c_int), ("outcomes", C.POINTER(Outcome)), ("outcome_drafts", C.POINTER(C.c_int)),
                ("n_trace", C.c_int), ("trace", C.POINTER(C.c_int)), ("hotness", C.POINTER(C.c_uint64)),
                ("tau_mean", C.c_double), ("tokens_total", C.c_uint64), ("phases", C.c_int),
                ("speculation_s", C.c_double), ("verification_s", C.c_double), ("modeled_seconds", C.c_double),
                ("tokens_per_sec", C.c_double),
                ("bytes_spec", C.c_uint64), ("bytes_verify", C.c_uint64), ("bytes_baseline", C.c_uint64),
                ("bytes_total", C.c_uint64), ("setup_bytes", C.c_uint64), ("warmup_bytes", C.c_uint64),
                ("lambda_", C.c_double), ("c_measured", C.c_double), ("wall_s", C.c_double), ("gpu_s", C.c_double),
                ("h2d_expert_bytes", C.c_uint64), ("h2d_s", C.c_double),
                ("prefetch_bytes", C.c_uint64), ("prefetch_wasted_bytes", C.c_uint64)]


_LIB = None


def build(quiet: bool = True) -> None:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    import subprocess
    root = os.path.dirname(HERE)
    subprocess.run(["make", "-s", "-j8", "-C", root], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise EngineError(3, f"{LIB_PATH} not built (run `make` or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, ip, dp, fp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_float)
    L.smoe_last_error.restype = C.c_char_p
    L.smoe_engine_create.argtypes = [C.POINTER(EngineConfig), C.POINTER(vp)]
    L.smoe_engine_destroy.argtypes = [vp]
    L.smoe_engine_info.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), ip]
    L.smoe_engine_stream.restype = vp
    L.smoe_engine_stream.argtypes = [vp]
    L.smoe_init_weights_exact.argtypes = [vp]
    L.smoe_init_weights_device.argtypes = [vp, C.c_uint64]
    L.smoe_upload_tensor.argtypes = [vp, C.c_char_p, C.c_int, C.c_int, dp, C.c_longlong]
    L.smoe_set_affinity.argtypes = [vp, dp]
    L.smoe_build_affinity_device.argtypes = [vp]
    L.smoe_get_affinity.argtypes = [vp, dp]
    L.smoe_forward.argtypes = [vp, ip, C.c_int, ip, C.c_int, C.c_int, fp, ip, ip]
    L.smoe_run_specmoe.argtypes = [vp, C.POINTER(RunConfig), ip, C.c_int, C.c_int, C.POINTER(C.POINTER(RunResultC))]
    L.smoe_run_ondemand.argtypes = [vp, C.POINTER(RunConfig), ip, C.c_int, C.c_int, C.POINTER(C.POINTER(RunResultC))]
    L.smoe_run_overlap.argtypes = [vp, C.POINTER(RunConfig), ip, C.c_int, C.c_int, C.POINTER(C.POINTER(RunResultC))]
    L.smoe_run_caching.argtypes = [vp, C.POINTER(RunConfig), C.c_double, ip, C.c_int, C.c_int,
                                   C.POINTER(C.POINTER(RunResultC))]
    L.smoe_free_result.argtypes = [C.POINTER(RunResultC)]
    L.smoe_spec_begin.argtypes = [vp, C.POINTER(RunConfig), ip, C.c_int, C.c_int]
    L.smoe_spec_step.argtypes = [vp, ip, ip]
    L.smoe_spec_end.argtypes = [vp, C.POINTER(C.POINTER(RunResultC))]
    L.smoe_counters.argtypes = [vp, C.POINTER(C.c_uint64), dp, dp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                C.c_int]
    L.smoe_bench_expert_gemm.argtypes = [vp, C.c_int, C.c_int, dp, dp, dp, dp]
    L.smoe_ep_nccl_unique_id.argtypes = [vp, C.c_int]
    L.smoe_ep_attach_nccl.argtypes = [vp, vp, C.c_int]
    L.smoe_ep_loopback_create.restype = vp
    L.smoe_ep_loopback_create.argtypes = [C.c_int]
    L.smoe_ep_loopback_destroy.argtypes = [vp]
    L.smoe_ep_attach_loopback.argtypes = [vp, vp]
    L.smoe_ep_attach_host.argtypes = [vp, HOST_ALLGATHER, vp]
    L.smoe_profile_reset.argtypes = [vp]
    L.smoe_profile_stop.argtypes = [vp]
    L.smoe_counter.argtypes = [vp, C.c_char_p, dp]
    L.smoe_profile_read.argtypes = [vp, C.c_char_p, dp, C.POINTER(C.c_longlong), dp]
    L.smoe_make_prompts.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, ip]
    _LIB = L
    return L


def _check(rc: int) -> None:
    if rc != 0:
        raise EngineError(rc, lib().smoe_last_error().decode(errors="replace"))


def make_prompts_native(seed: int, batch: int, prompt_len: int, vocab: int) -> list[list[int]]:
    """The harness's make_prompts (C++, harness.cpp) through the C ABI; host only."""
    out = (C.c_int * max(1, batch * prompt_len))()
    _check(lib().smoe_make_prompts(seed, batch, prompt_len, vocab, out))
    return [list(out[b * prompt_len:(b + 1) * prompt_len]) for b in range(batch)]


@dataclass
class ModelSpec:
    """specmoe::ModelSpec (model.hpp:16-32) + the expert form."""
    num_layers: int = 4
    experts: int = 16
    top_k: int = 2
    hidden: int = 32
    ffn: int = 64
    vocab: int = 64
    gate_skew: float = 0.0
    seed: int = 0
    moe_mask: list | None = None
    expert_kind: int = TANH2
    # extension: attn_heads > 0 = real GQA attention with RoPE and a paged KV cache in
    # place of the reference's prefix-mean + mix surrogate (restated in oracle/specmoe_oracle.c fwd_attn)
    attn_heads: int = 0
    kv_heads: int = 0
    head_dim: int = 0
    rope_theta: float = 10000.0

    @property
    def moe_layers(self) -> int:
        return self.num_layers if self.moe_mask is None else int(sum(1 for m in self.moe_mask if m))

    def bytes_per_expert(self) -> int:  # memsim.cpp:17-20 (reference accounting units)
        return 2 * self.hidden * self.ffn * 4


@dataclass
class RunCfg:
    gamma: int = 10
    n_draft: int = 4
    max_new_tokens: int = 32
    use_affinity: bool = True
    warmup_steps: int = 64
    policy: str = "hot_temporal"
    collect_trace: bool = False
    run_seed: int = 0
    device_capacity_bytes: int = 0
    bytes_per_expert: int = 0
    host_bandwidth: float = 64e9
    ssd_bandwidth: float = 0.0
    compute_rate: float = 1e6
    compute_cost_per_expert: float = 2e-6
    mode: str = "greedy"       # "greedy" | "sampling" (DecodeMode, specdec.hpp:15)
    temperature: float = 1.0

    def to_c(self, spec: ModelSpec) -> RunConfig:
        bpe = self.bytes_per_expert or spec.bytes_per_expert()
        cap = self.device_capacity_bytes or spec.moe_layers * spec.experts * bpe
        return RunConfig(self.gamma, self.n_draft, self.max_new_tokens, int(self.use_affinity), self.warmup_steps,
                         POLICIES[self.policy], int(self.collect_trace), self.run_seed, cap, bpe, self.host_bandwidth,
                         self.ssd_bandwidth, self.compute_rate, self.compute_cost_per_expert,
                         {"greedy": 0, "sampling": 1}[self.mode], self.temperature)


class Ledger(Sequence):
    """The run's expert-residency ledger (ledger.hpp LedgerEntry list): (phase, step, layer, expert, bytes)
    tuples, built on access from one copied record array (a B=32 run of 128 tokens per sequence carries
    ~10^5 entries; turning them all into Python tuples up front cost ~20 ms of the run's wall time)."""

    def __init__(self, rec=None):
        self._rec = rec if rec is not None else np.zeros(0, dtype=LEDGER_DTYPE)
        self._list = None

    def _tuples(self) -> list:
        if self._list is None:
            lv = self._rec
            self._list = list(zip([PHASES[x] for x in lv["phase"].tolist()], lv["step"].tolist(),
                                  lv["layer"].tolist(), lv["expert"].tolist(), lv["bytes"].tolist()))
        return self._list

    def __len__(self) -> int:
        return len(self._rec)

    def __getitem__(self, i):
        return self._tuples()[i]

    def __iter__(self):
        return iter(self._tuples())

    def __eq__(self, other) -> bool:
        if isinstance(other, Ledger):
            return len(self) == len(other) and bool(np.array_equal(self._rec, other._rec))
        if isinstance(other, (list, tuple)):
            return self._tuples() == list(other)
        return NotImplemented

    def __repr__(self) -> str:
        return f"Ledger({self._tuples()!r})"


@dataclass
class RunResult:
    tokens: list
    ledger: Ledger = field(default_factory=Ledger)
    outcomes: list = field(default_factory=list)
    trace: list = field(default_factory=list)
    hotness: np.ndarray | None = None
    metrics: dict = field(default_factory=dict)


def _view(ptr, n, shape=None):
    """numpy view of n elements behind a ctypes pointer (empty for n == 0 / NULL)."""
    if n <= 0 or not ptr:
        return np.zeros(0 if shape is None else (0,) + tuple(shape[1:]), dtype=np.int64)
    a = np.ctypeslib.as_array(ptr, shape=(n,))
    return a if shape is None else a.reshape(shape)


def _collect(rp) -> RunResult:
    """Flatten the C result into Python values (whole arrays at a time: a B=64 run_specmoe of 128 tokens
    carries ~30k ledger entries, whose per-element ctypes reads cost ~0.1 s)."""
    r = rp.contents
    try:
        ntok = _view(r.n_tokens, r.B)
        tok = _view(r.tokens, r.B * r.max_new, (r.B, r.max_new)) if r.B * r.max_new else None
        toks = [tok[b, :ntok[b]].tolist() if tok is not None else [] for b in range(r.B)]
        led = Ledger(_view(r.ledger, r.n_ledger).copy() if r.n_ledger else None)
        g = r.gamma
        ov = _view(r.outcomes, r.n_outcomes)
        if r.n_outcomes:
            dr = _view(r.outcome_drafts, r.n_outcomes * g, (r.n_outcomes, g)).tolist() if g else [[]] * r.n_outcomes
            outc = list(zip(ov["seq"].tolist(), ov["phase"].tolist(), ov["accepted"].tolist(), ov["correction"].tolist(),
                            ov["tokens_generated"].tolist(), [tuple(x) for x in dr]))
        else:
            outc = []
        K = r.top_k
        if r.n_trace:
            tv = _view(r.trace, r.n_trace * (3 + K), (r.n_trace, 3 + K)).tolist()
            tr = [(x[0], x[1], x[2], tuple(x[3:])) for x in tv]
        else:
            tr = []
        hot = np.array(_view(r.hotness, r.moe_layers * r.experts), dtype=np.uint64)
        met = {k: getattr(r, k) for k in ("tau_mean", "tokens_total", "phases", "speculation_s", "verification_s",
                                          "modeled_seconds", "tokens_per_sec", "bytes_spec", "bytes_verify",
                                          "bytes_baseline", "bytes_total", "setup_bytes", "warmup_bytes",
                                          "c_measured", "wall_s", "gpu_s", "h2d_expert_bytes", "h2d_s",
                                          "prefetch_bytes", "prefetch_wasted_bytes")}
        met["lambda"] = r.lambda_
        return RunResult(toks, led, outc, tr, hot.reshape(r.moe_layers, r.experts), met)
    finally:
        lib().smoe_free_result(rp)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(256)
    n = lib().smoe_ep_nccl_unique_id(buf, 256)
    if n <= 0:
        raise EngineError(-n if n < 0 else 3, lib().smoe_last_error().decode(errors="replace"))
    return buf.raw[:n]


# int (*)(void* user, const void* send, void* recv, uint64_t bytes) -- include/specmoe_b200.h
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)


class HostTransport:
    """One process per EP rank; the engine's collectives go through `allgather(data: bytes) -> list[bytes]`
    (rank order), e.g. a torch.distributed gloo all-gather.  The fused exchange's peer buffers are CUDA
    IPC handles all-gathered the same way, so ranks may share one GPU."""

    def __init__(self, allgather):
        self._fn = allgather

        def cb(user, send, recv, nbytes):
            try:
                parts = self._fn(C.string_at(send, nbytes))
                for r, blob in enumerate(parts):
                    if len(blob) != nbytes:
                        return 2
                    C.memmove(recv + r * nbytes, blob, nbytes)
                return 0
            except Exception:  # never unwind through the C++ engine
                import traceback
                traceback.print_exc()
                return 1
        self.cfunc = HOST_ALLGATHER(cb)  # kept alive as long as the transport


def gloo_allgather(group=None):
    """A HostTransport all-gather over torch.distributed (any backend with CPU tensors, e.g. gloo)."""
    import torch
    import torch.distributed as dist

    def ag(data: bytes):
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(out, t, group=group)
        return [o.numpy().tobytes() for o in out]
    return ag


class LoopbackGroup:
    """G virtual EP ranks on one device (each rank: an Engine driven by its own thread)."""

    def __init__(self, world: int):
        self.h = lib().smoe_ep_loopback_create(world)
        if not self.h:
            raise EngineError(1, lib().smoe_last_error().decode(errors="replace"))

    def close(self):
        if self.h:
            lib().smoe_ep_loopback_destroy(self.h)
            self.h = None


def _iarr(x):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int32))
    return a, a.ctypes.data_as(C.POINTER(C.c_int))


class Engine:
    """One B200 engine: device-resident weights + state for one model (specmoe::ModelWeights analogue)."""

    def __init__(self, spec: ModelSpec, weight_type: int = F32, max_batch: int = 8, max_gamma: int = 10,
                 gemm: int = GEMM_AUTO, device: int = 0, offload: int = 0, hbm_expert_slots: int = 0,
                 ep_rank: int = 0, ep_world: int = 1, max_seq_len: int = 0):
        self.spec = spec
        L = lib()
        self._mask = None
        if spec.moe_mask is not None:
            self._mask = (C.c_uint8 * spec.num_layers)(*[1 if m else 0 for m in spec.moe_mask])
        cfg = EngineConfig(spec.num_layers, spec.experts, spec.top_k, spec.hidden, spec.ffn, spec.vocab, spec.gate_skew,
                           spec.seed, C.cast(self._mask, C.POINTER(C.c_uint8)) if self._mask is not None else None,
                           spec.expert_kind, weight_type, max_batch, max_gamma, gemm, device, offload,
                           hbm_expert_slots, ep_rank, ep_world, spec.attn_heads, spec.kv_heads, spec.head_dim,
                           spec.rope_theta, max_seq_len)
        h = C.c_void_p()
        _check(L.smoe_engine_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().smoe_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().smoe_engine_stream(self.h) or 0

    def info(self):
        db, bpe, m = C.c_uint64(), C.c_uint64(), C.c_int()
        _check(lib().smoe_engine_info(self.h, C.byref(db), C.byref(bpe), C.byref(m)))
        return {"device_bytes_used": db.value, "bytes_per_expert": bpe.value, "moe_layers": m.value}

    # ---- weights (model.cpp:106-143) and affinity (drafting.cpp:28-57)
    def init_exact(self):
        _check(lib().smoe_init_weights_exact(self.h))
        return self

    def init_device(self, seed: int = 0):
        _check(lib().smoe_init_weights_device(self.h, seed))
        return self

    def upload(self, name: str, tensor, layer: int = -1, expert: int = -1):
        t = np.ascontiguousarray(np.asarray(tensor, dtype=np.float64))
        _check(lib().smoe_upload_tensor(self.h, name.encode(), layer, expert, t.ctypes.data_as(C.POINTER(C.c_double)),
                                        t.size))

    def build_affinity_device(self):
        _check(lib().smoe_build_affinity_device(self.h))

    def set_affinity(self, dist):
        D = np.ascontiguousarray(np.asarray(dist, dtype=np.float64))
        _check(lib().smoe_set_affinity(self.h, D.ctypes.data_as(C.POINTER(C.c_double))))

    def affinity(self) -> np.ndarray:
        M, E = self.spec.moe_layers, self.spec.experts
        out = np.empty(M * E * E, dtype=np.float64)
        _check(lib().smoe_get_affinity(self.h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out.reshape(M, E, E)

    # ---- forward (model.hpp:114-116)
    def forward(self, prefix, restricted=None, use_affinity=False):
        sp = self.spec
        p, pp = _iarr(prefix)
        rp, nd = None, 0
        if restricted is not None:
            r = np.asarray(restricted, dtype=np.int32)
            nd = r.shape[1]
            r, rp = _iarr(r.reshape(-1))
        logits = np.empty(sp.vocab, dtype=np.float32)
        raw = np.zeros(sp.moe_layers * sp.top_k, dtype=np.int32)
        fin = np.zeros_like(raw)
        _check(lib().smoe_forward(self.h, pp, len(p), rp, nd, int(use_affinity),
                                  logits.ctypes.data_as(C.POINTER(C.c_float)), raw.ctypes.data_as(C.POINTER(C.c_int)),
                                  fin.ctypes.data_as(C.POINTER(C.c_int))))
        return logits, raw.reshape(sp.moe_layers, sp.top_k), fin.reshape(sp.moe_layers, sp.top_k)

    # ---- loops (specdec.hpp:122-124, baselines.hpp:24-26)
    def run_specmoe(self, cfg: RunCfg, prompts) -> RunResult:
        P = np.asarray(prompts, dtype=np.int32)
        c = cfg.to_c(self.spec)
        p, pp = _iarr(P.reshape(-1))
        out = C.POINTER(RunResultC)()
        _check(lib().smoe_run_specmoe(self.h, C.byref(c), pp, P.shape[0], P.shape[1], C.byref(out)))
        return _collect(out)

    def run_ondemand(self, cfg: RunCfg, prompts) -> RunResult:
        P = np.asarray(prompts, dtype=np.int32)
        c = cfg.to_c(self.spec)
        p, pp = _iarr(P.reshape(-1))
        out = C.POINTER(RunResultC)()
        _check(lib().smoe_run_ondemand(self.h, C.byref(c), pp, P.shape[0], P.shape[1], C.byref(out)))
        return _collect(out)

    def run_overlap(self, cfg: RunCfg, prompts) -> RunResult:
        """baselines.hpp:30-34 on the physical store (next-layer prefetch overlapping each layer)."""
        P = np.asarray(prompts, dtype=np.int32)
        c = cfg.to_c(self.spec)
        p, pp = _iarr(P.reshape(-1))
        out = C.POINTER(RunResultC)()
        _check(lib().smoe_run_overlap(self.h, C.byref(c), pp, P.shape[0], P.shape[1], C.byref(out)))
        return _collect(out)

    def run_caching(self, cfg: RunCfg, prompts, cache_fraction: float = 0.10) -> RunResult:
        """baselines.hpp:36-41: top ceil(cache_fraction*E) hot experts per layer pinned, then on-demand."""
        P = np.asarray(prompts, dtype=np.int32)
        c = cfg.to_c(self.spec)
        p, pp = _iarr(P.reshape(-1))
        out = C.POINTER(RunResultC)()
        _check(lib().smoe_run_caching(self.h, C.byref(c), cache_fraction, pp, P.shape[0], P.shape[1], C.byref(out)))
        return _collect(out)

    # ---- stepped loop (bench)
    def spec_begin(self, cfg: RunCfg, prompts):
        P = np.asarray(prompts, dtype=np.int32)
        self._c = cfg.to_c(self.spec)
        self._p, pp = _iarr(P.reshape(-1))
        _check(lib().smoe_spec_begin(self.h, C.byref(self._c), pp, P.shape[0], P.shape[1]))

    def spec_step(self):
        tok, act = C.c_int(), C.c_int()
        _check(lib().smoe_spec_step(self.h, C.byref(tok), C.byref(act)))
        return tok.value, act.value

    def spec_end(self) -> RunResult:
        out = C.POINTER(RunResultC)()
        _check(lib().smoe_spec_end(self.h, C.byref(out)))
        return _collect(out)

    # ---- expert parallelism
    def attach_nccl(self, unique_id: bytes):
        buf = C.create_string_buffer(unique_id, len(unique_id))
        _check(lib().smoe_ep_attach_nccl(self.h, buf, len(unique_id)))

    def attach_host(self, transport: "HostTransport"):
        self._transport = transport  # the callback must outlive the engine's use of it
        _check(lib().smoe_ep_attach_host(self.h, transport.cfunc, None))

    def attach_loopback(self, group: "LoopbackGroup"):
        _check(lib().smoe_ep_attach_loopback(self.h, group.h))

    def counters(self, reset: bool = False) -> dict:
        la, h2d, d2h = C.c_uint64(), C.c_uint64(), C.c_uint64()
        eb, db = C.c_double(), C.c_double()
        _check(lib().smoe_counters(self.h, C.byref(la), C.byref(eb), C.byref(db), C.byref(h2d), C.byref(d2h),
                                   int(reset)))
        return {"launches": la.value, "alg_expert_bytes": eb.value, "alg_dense_bytes": db.value,
                "ctl_h2d": h2d.value, "ctl_d2h": d2h.value}

    def bench_expert_gemm(self, T: int, iters: int = 10) -> dict:
        u, d, bu, bd = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        _check(lib().smoe_bench_expert_gemm(self.h, T, iters, C.byref(u), C.byref(d), C.byref(bu), C.byref(bd)))
        return {"up_ms": u.value, "down_ms": d.value, "up_bytes": bu.value, "down_bytes": bd.value,
                "up_GBps": bu.value / (u.value * 1e-3) / 1e9 if u.value else 0.0,
                "down_GBps": bd.value / (d.value * 1e-3) / 1e9 if d.value else 0.0}

    def profile_reset(self):
        _check(lib().smoe_profile_reset(self.h))

    def counter(self, name: str) -> float:
        v = C.c_double()
        _check(lib().smoe_counter(self.h, name.encode(), C.byref(v)))
        return v.value

    def profile_stop(self):
        _check(lib().smoe_profile_stop(self.h))

    def profile_read(self, cls: str):
        ms, n, by = C.c_double(), C.c_longlong(), C.c_double()
        _check(lib().smoe_profile_read(self.h, cls.encode(), C.byref(ms), C.byref(n), C.byref(by)))
        return {"ms": ms.value, "launches": n.value, "bytes": by.value}
