"""oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes bindings for the two CPU oracles that share oracle/oracle_abi.h:

* ``Oracle("ref")``  -> oracle/_ref/libspecmoe_ref.so, the reference's own C++ sources
  (/root/reference/proj/core/src) compiled by oracle/Makefile plus a type adapter;
* ``Oracle("port")`` -> oracle/liboracle_port.so, the plain-C restatement
  (oracle/specmoe_oracle.c), which also carries the swiglu3 extension.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this module.  The product (paper_2604_10152_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libspecmoe_ref.so"),
    "port": os.path.join(HERE, "liboracle_port.so"),
}
REF_SRC = "/root/reference/proj/core/src"

POLICIES = {"random": 0, "hot_global": 1, "hot_temporal": 2}
PHASES = {0: "speculation", 1: "verification", 2: "baseline-step"}


class OmSpec(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("experts", C.c_int), ("top_k", C.c_int), ("hidden", C.c_int),
                ("ffn", C.c_int), ("vocab", C.c_int), ("gate_skew", C.c_double), ("seed", C.c_uint64),
                ("moe_mask", C.POINTER(C.c_uint8)), ("expert_kind", C.c_int), ("attn_heads", C.c_int),
                ("kv_heads", C.c_int), ("head_dim", C.c_int), ("rope_theta", C.c_double)]


class OmRunCfg(C.Structure):
    _fields_ = [("gamma", C.c_int), ("n_draft", C.c_int), ("max_new_tokens", C.c_int), ("use_affinity", C.c_int),
                ("warmup_steps", C.c_int), ("policy", C.c_int), ("collect_trace", C.c_int), ("run_seed", C.c_uint64),
                ("device_capacity_bytes", C.c_uint64), ("bytes_per_expert", C.c_uint64),
                ("host_bandwidth", C.c_double), ("ssd_bandwidth", C.c_double), ("compute_rate", C.c_double),
                ("compute_cost_per_expert", C.c_double)]


class OmLedger(C.Structure):
    _fields_ = [("phase", C.c_int), ("step", C.c_int), ("layer", C.c_int), ("expert", C.c_int), ("bytes", C.c_uint64)]


class OmOutcome(C.Structure):
    _fields_ = [("seq", C.c_int), ("phase", C.c_int), ("accepted", C.c_int), ("correction", C.c_int),
                ("tokens_generated", C.c_int)]


class OmResult(C.Structure):
    _fields_ = [("B", C.c_int), ("max_new", C.c_int), ("moe_layers", C.c_int), ("experts", C.c_int),
                ("top_k", C.c_int), ("gamma", C.c_int),
                ("tokens", C.POINTER(C.c_int)), ("n_tokens", C.POINTER(C.c_int)),
                ("n_ledger", C.c_int), ("ledger", C.POINTER(OmLedger)),
                ("n_outcomes", C.c_int), ("outcomes", C.POINTER(OmOutcome)), ("outcome_drafts", C.POINTER(C.c_int)),
                ("n_trace", C.c_int), ("trace", C.POINTER(C.c_int)), ("hotness", C.POINTER(C.c_uint64)),
                ("tau_mean", C.c_double), ("tokens_total", C.c_uint64), ("phases", C.c_int),
                ("speculation_s", C.c_double), ("verification_s", C.c_double), ("modeled_seconds", C.c_double),
                ("tokens_per_sec", C.c_double),
                ("bytes_spec", C.c_uint64), ("bytes_verify", C.c_uint64), ("bytes_baseline", C.c_uint64),
                ("bytes_total", C.c_uint64), ("setup_bytes", C.c_uint64), ("warmup_bytes", C.c_uint64),
                ("lambda_", C.c_double), ("c_measured", C.c_double), ("wall_s", C.c_double)]


def build_oracles(which=("port", "ref")) -> None:
    """Compile the oracle libraries (gcc/g++ only; the reference only where its sources exist)."""
    targets = [t for t in which if t == "port" or os.path.isdir(REF_SRC)]
    if targets:
        subprocess.run(["make", "-s", "-C", HERE] + list(targets), check=True)


@dataclass
class ModelSpec:
    """Mirror of specmoe::ModelSpec (model.hpp:16-32) plus the port-only expert_kind."""
    num_layers: int = 4
    experts: int = 16
    top_k: int = 2
    hidden: int = 32
    ffn: int = 64
    vocab: int = 64
    gate_skew: float = 0.0
    seed: int = 0
    moe_mask: list | None = None
    expert_kind: int = 0  # 0 tanh2, 1 swiglu3
    attn_heads: int = 0   # > 0: real GQA attention with RoPE instead of the prefix-mean surrogate (port only)
    kv_heads: int = 0
    head_dim: int = 0
    rope_theta: float = 10000.0

    @property
    def moe_layers(self) -> int:
        return self.num_layers if self.moe_mask is None else int(sum(1 for m in self.moe_mask if m))

    def bytes_per_expert(self) -> int:  # memsim.cpp:17-20
        return 2 * self.hidden * self.ffn * 4


@dataclass
class RunCfg:
    """SpecConfig (specdec.hpp:17-29) + TierConfig (memsim.hpp:28-39) + policy + seed (greedy only)."""
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

    def for_spec(self, spec: ModelSpec) -> "RunCfg":
        """Fill bytes_per_expert and (if 0) a capacity that holds every expert of the model."""
        c = RunCfg(**self.__dict__)
        if c.bytes_per_expert == 0:
            c.bytes_per_expert = spec.bytes_per_expert()
        if c.device_capacity_bytes == 0:
            c.device_capacity_bytes = spec.moe_layers * spec.experts * c.bytes_per_expert
        return c


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class RunResult:
    tokens: list
    ledger: list = field(default_factory=list)  # (phase_name, step, layer, expert, bytes)
    outcomes: list = field(default_factory=list)  # (seq, phase, accepted, correction, generated, drafts)
    trace: list = field(default_factory=list)     # (step, seq, layer, experts tuple)
    hotness: np.ndarray | None = None
    metrics: dict = field(default_factory=dict)


class Oracle:
    def __init__(self, kind: str = "ref"):
        path = LIBS[kind]
        if not os.path.exists(path):
            build_oracles((kind,))
        self.kind = kind
        self.lib = L = C.CDLL(path)
        vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
        L.om_build_model.restype = vp
        L.om_build_model.argtypes = [C.POINTER(OmSpec), C.c_char_p, C.c_int]
        L.om_free_model.argtypes = [vp]
        L.om_get_tensor.restype = C.c_longlong
        L.om_get_tensor.argtypes = [vp, C.c_char_p, C.c_int, C.c_int, dp, C.c_longlong]
        L.om_build_affinity.restype = vp
        L.om_build_affinity.argtypes = [vp]
        L.om_free_affinity.argtypes = [vp]
        L.om_affinity_get.argtypes = [vp, dp, C.c_longlong]
        L.om_forward.argtypes = [vp, ip, C.c_int, ip, C.c_int, vp, dp, ip, ip, C.c_char_p, C.c_int]
        L.om_run_specmoe.restype = C.POINTER(OmResult)
        L.om_run_specmoe.argtypes = [vp, C.POINTER(OmRunCfg), ip, C.c_int, C.c_int, vp, C.c_char_p, C.c_int]
        L.om_run_ondemand.restype = C.POINTER(OmResult)
        L.om_run_ondemand.argtypes = [vp, C.POINTER(OmRunCfg), ip, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.om_run_overlap.restype = C.POINTER(OmResult)
        L.om_run_overlap.argtypes = [vp, C.POINTER(OmRunCfg), ip, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.om_run_caching.restype = C.POINTER(OmResult)
        L.om_run_caching.argtypes = [vp, C.POINTER(OmRunCfg), C.c_double, ip, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.om_free_result.argtypes = [C.POINTER(OmResult)]
        L.om_route_topk.argtypes = [dp, C.c_int, C.c_int, ip]
        L.om_greedy_next.argtypes = [dp, C.c_int]
        L.om_softmax.argtypes = [dp, C.c_int, dp]
        L.om_nearest_draft_expert.argtypes = [dp, C.c_int, C.c_int, ip, C.c_int, ip, C.c_int]
        L.om_select_draft_experts.argtypes = [C.c_int, C.POINTER(C.c_uint64), C.c_int, C.c_int, ip, C.c_int,
                                              C.c_uint64, ip]
        L.om_time_forward.restype = C.c_double
        L.om_time_forward.argtypes = [vp, ip, C.c_int, C.c_int, C.c_int]
        L.om_skewness.restype = C.c_double
        L.om_skewness.argtypes = [C.POINTER(C.c_uint64), C.c_int, C.c_int, C.c_uint64, C.c_double]

    # ---------------------------------------------------------------- model
    def build(self, spec: ModelSpec) -> "OracleModel":
        mask = None
        if spec.moe_mask is not None:
            mask = (C.c_uint8 * spec.num_layers)(*[1 if m else 0 for m in spec.moe_mask])
        s = OmSpec(spec.num_layers, spec.experts, spec.top_k, spec.hidden, spec.ffn, spec.vocab, spec.gate_skew,
                   spec.seed, C.cast(mask, C.POINTER(C.c_uint8)) if mask is not None else None, spec.expert_kind,
                   spec.attn_heads, spec.kv_heads, spec.head_dim, spec.rope_theta)
        err = C.create_string_buffer(256)
        h = self.lib.om_build_model(C.byref(s), err, 256)
        if not h:
            raise OracleError(1, err.value.decode())
        return OracleModel(self, h, spec)


def _iarr(x):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int32))
    return a, a.ctypes.data_as(C.POINTER(C.c_int))


class OracleModel:
    def __init__(self, oracle: Oracle, handle, spec: ModelSpec):
        self.o, self.h, self.spec = oracle, handle, spec
        self._aff = None

    def __del__(self):
        try:
            if self._aff:
                self.o.lib.om_free_affinity(self._aff)
            if self.h:
                self.o.lib.om_free_model(self.h)
        except Exception:
            pass

    def tensor(self, name: str, layer: int = -1, expert: int = -1) -> np.ndarray:
        n = self.o.lib.om_get_tensor(self.h, name.encode(), layer, expert, None, 0)
        if n < 0:
            raise KeyError((name, layer, expert))
        out = np.empty(n, dtype=np.float64)
        self.o.lib.om_get_tensor(self.h, name.encode(), layer, expert,
                                 out.ctypes.data_as(C.POINTER(C.c_double)), n)
        return out

    def affinity(self) -> np.ndarray:
        if not self._aff:
            self._aff = self.o.lib.om_build_affinity(self.h)
        M, E = self.spec.moe_layers, self.spec.experts
        out = np.empty(M * E * E, dtype=np.float64)
        self.o.lib.om_affinity_get(self._aff, out.ctypes.data_as(C.POINTER(C.c_double)), out.size)
        return out.reshape(M, E, E)

    def forward(self, prefix, restricted=None, use_affinity=False):
        sp = self.spec
        p, pp = _iarr(prefix)
        rp, nd = None, 0
        if restricted is not None:
            r = np.asarray(restricted, dtype=np.int32)
            nd = r.shape[1]
            r, rp = _iarr(r.reshape(-1))
        aff = None
        if use_affinity:
            self.affinity()
            aff = self._aff
        logits = np.empty(sp.vocab, dtype=np.float64)
        raw = np.zeros(sp.moe_layers * sp.top_k, dtype=np.int32)
        fin = np.zeros_like(raw)
        err = C.create_string_buffer(256)
        rc = self.o.lib.om_forward(self.h, pp, len(p), rp, nd, aff, logits.ctypes.data_as(C.POINTER(C.c_double)),
                                   raw.ctypes.data_as(C.POINTER(C.c_int)), fin.ctypes.data_as(C.POINTER(C.c_int)),
                                   err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return logits, raw.reshape(sp.moe_layers, sp.top_k), fin.reshape(sp.moe_layers, sp.top_k)

    def forward_gates(self, prefix):
        """Port only: (logits [V], gate logits + bias [moe_layers][E]) of one forward."""
        sp = self.spec
        p, pp = _iarr(prefix)
        lg = np.empty(sp.vocab, dtype=np.float64)
        gates = np.empty(sp.moe_layers * sp.experts, dtype=np.float64)
        err = C.create_string_buffer(256)
        f = self.o.lib.om_forward_gates
        f.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                      C.c_char_p, C.c_int]
        rc = f(self.h, pp, len(p), lg.ctypes.data_as(C.POINTER(C.c_double)),
               gates.ctypes.data_as(C.POINTER(C.c_double)), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return lg, gates.reshape(sp.moe_layers, sp.experts)

    def time_forward(self, prefix, threads: int = 1, iters: int = 1) -> float:
        """Wall seconds for `threads` concurrent threads x `iters` forward() calls each."""
        p, pp = _iarr(prefix)
        t = self.o.lib.om_time_forward(self.h, pp, len(p), threads, iters)
        if t < 0:
            raise OracleError(2, "time_forward failed")
        return t

    # ---------------------------------------------------------------- loops
    def _cfg(self, cfg: RunCfg) -> OmRunCfg:
        c = cfg.for_spec(self.spec)
        return OmRunCfg(c.gamma, c.n_draft, c.max_new_tokens, int(c.use_affinity), c.warmup_steps,
                        POLICIES[c.policy], int(c.collect_trace), c.run_seed, c.device_capacity_bytes,
                        c.bytes_per_expert, c.host_bandwidth, c.ssd_bandwidth, c.compute_rate,
                        c.compute_cost_per_expert)

    def run_specmoe(self, cfg: RunCfg, prompts) -> RunResult:
        P = np.asarray(prompts, dtype=np.int32)
        c = self._cfg(cfg)
        aff = None
        if cfg.use_affinity:
            self.affinity()
            aff = self._aff
        p, pp = _iarr(P.reshape(-1))
        err = C.create_string_buffer(256)
        r = self.o.lib.om_run_specmoe(self.h, C.byref(c), pp, P.shape[0], P.shape[1], aff, err, 256)
        return self._collect(r, err)

    def run_ondemand(self, cfg: RunCfg, prompts) -> RunResult:
        P = np.asarray(prompts, dtype=np.int32)
        c = self._cfg(cfg)
        p, pp = _iarr(P.reshape(-1))
        err = C.create_string_buffer(256)
        r = self.o.lib.om_run_ondemand(self.h, C.byref(c), pp, P.shape[0], P.shape[1], err, 256)
        return self._collect(r, err)

    def run_overlap(self, cfg: RunCfg, prompts) -> RunResult:
        P = np.asarray(prompts, dtype=np.int32)
        c = self._cfg(cfg)
        p, pp = _iarr(P.reshape(-1))
        err = C.create_string_buffer(256)
        r = self.o.lib.om_run_overlap(self.h, C.byref(c), pp, P.shape[0], P.shape[1], err, 256)
        return self._collect(r, err)

    def run_caching(self, cfg: RunCfg, prompts, cache_fraction: float = 0.10) -> RunResult:
        """run_caching with BaselineConfig{caching, cache_fraction, warmup_steps = cfg.warmup_steps}."""
        P = np.asarray(prompts, dtype=np.int32)
        c = self._cfg(cfg)
        p, pp = _iarr(P.reshape(-1))
        err = C.create_string_buffer(256)
        r = self.o.lib.om_run_caching(self.h, C.byref(c), cache_fraction, pp, P.shape[0], P.shape[1], err, 256)
        return self._collect(r, err)

    def _collect(self, rp, err) -> RunResult:
        if not rp:
            msg = err.value.decode()
            raise OracleError(1 if "violated" in msg or "capacity below" in msg else 2, msg)
        r = rp.contents
        try:
            toks = [[r.tokens[b * r.max_new + i] for i in range(r.n_tokens[b])] for b in range(r.B)]
            led = [(PHASES[r.ledger[i].phase], r.ledger[i].step, r.ledger[i].layer, r.ledger[i].expert,
                    r.ledger[i].bytes) for i in range(r.n_ledger)]
            g = r.gamma
            outc = [(r.outcomes[i].seq, r.outcomes[i].phase, r.outcomes[i].accepted, r.outcomes[i].correction,
                     r.outcomes[i].tokens_generated, tuple(r.outcome_drafts[i * g + j] for j in range(g)))
                    for i in range(r.n_outcomes)]
            K = r.top_k
            tr = [(r.trace[i * (3 + K)], r.trace[i * (3 + K) + 1], r.trace[i * (3 + K) + 2],
                   tuple(r.trace[i * (3 + K) + 3 + k] for k in range(K))) for i in range(r.n_trace)]
            hot = np.array([r.hotness[i] for i in range(r.moe_layers * r.experts)], dtype=np.uint64)
            hot = hot.reshape(r.moe_layers, r.experts)
            met = {k: getattr(r, k) for k in ("tau_mean", "tokens_total", "phases", "speculation_s",
                                              "verification_s", "modeled_seconds", "tokens_per_sec", "bytes_spec",
                                              "bytes_verify", "bytes_baseline", "bytes_total", "setup_bytes",
                                              "warmup_bytes", "c_measured", "wall_s")}
            met["lambda"] = r.lambda_
            return RunResult(toks, led, outc, tr, hot, met)
        finally:
            self.o.lib.om_free_result(rp)


# ---------------------------------------------------------------- primitives (SPEC KATs)
def route_topk(o: Oracle, logits, k):
    x = np.ascontiguousarray(np.asarray(logits, dtype=np.float64))
    out = np.zeros(k, dtype=np.int32)
    rc = o.lib.om_route_topk(x.ctypes.data_as(C.POINTER(C.c_double)), len(x), k,
                             out.ctypes.data_as(C.POINTER(C.c_int)))
    if rc:
        raise OracleError(-rc, "route_topk")
    return out.tolist()


def greedy_next(o: Oracle, logits):
    x = np.ascontiguousarray(np.asarray(logits, dtype=np.float64))
    rc = o.lib.om_greedy_next(x.ctypes.data_as(C.POINTER(C.c_double)), len(x))
    if rc < 0:
        raise OracleError(-rc, "greedy_next")
    return rc


def softmax(o: Oracle, logits):
    x = np.ascontiguousarray(np.asarray(logits, dtype=np.float64))
    out = np.zeros_like(x)
    rc = o.lib.om_softmax(x.ctypes.data_as(C.POINTER(C.c_double)), len(x), out.ctypes.data_as(C.POINTER(C.c_double)))
    if rc:
        raise OracleError(-rc, "softmax")
    return out


def nearest_draft_expert(o: Oracle, dist, raw, draft, excluded=()):
    D = np.ascontiguousarray(np.asarray(dist, dtype=np.float64))
    E = D.shape[0]
    d, dp = _iarr(list(draft) or [0])
    x, xp = _iarr(list(excluded) or [0])
    rc = o.lib.om_nearest_draft_expert(D.ctypes.data_as(C.POINTER(C.c_double)), E, raw, dp, len(draft), xp,
                                       len(excluded))
    if rc < 0:
        raise OracleError(-rc, "nearest_draft_expert")
    return rc


def select_draft_experts(o: Oracle, policy, counts, n_draft, current=None, seed=0):
    Cn = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    layers, E = Cn.shape
    cur = None
    if current is not None:
        cur_a, cur = _iarr(np.asarray(current).reshape(-1))
    out = np.zeros(layers * n_draft, dtype=np.int32)
    rc = o.lib.om_select_draft_experts(POLICIES[policy], Cn.ctypes.data_as(C.POINTER(C.c_uint64)), layers, E, cur,
                                       n_draft, seed, out.ctypes.data_as(C.POINTER(C.c_int)))
    if rc:
        raise OracleError(-rc, "select_draft_experts")
    return out.reshape(layers, n_draft).tolist()


def skewness(o: Oracle, counts, routed, top_fraction=0.25):
    Cn = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    return o.lib.om_skewness(Cn.ctypes.data_as(C.POINTER(C.c_uint64)), Cn.shape[0], Cn.shape[1], routed, top_fraction)
