"""ctypes binding of include/moa_b200.h (the reference-facing C-ABI).

This is the same binding a Python caller of the reference path would add
(INTEGRATION.md); the tests and bench.py drive the B200 path only through it.
There is no fallback: if libmoa_b200.so is missing or the GPU is absent the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import configs as _configs

LIB_PATH = Path(__file__).resolve().parent / "libmoa_b200.so"

MOA_OK, MOA_ERR_VALIDATION, MOA_ERR_RUNTIME, MOA_ERR_DEVICE, MOA_ERR_UNSUPPORTED = 0, 2, 3, 4, 5
MOA_ERR_PROVIDER_TRANSPORT, MOA_ERR_PROVIDER_CREDENTIALS, MOA_ERR_PROVIDER_BAD_RESPONSE = 6, 7, 8
MODES = {"sequential-pd": 0, "dp-only": 1, "dp-chunked-prefill": 2, "incremental-overlap": 3}
EVENT_KINDS = {1: "chunk", 2: "decode_end", 3: "cancel", 4: "reclaim"}


class ValidationError(Exception):
    """MOA_ERR_VALIDATION -- the reference's ValidationError (errors.hpp:10-13)."""


class RunError(Exception):
    """MOA_ERR_RUNTIME -- the reference's RunError (errors.hpp:17-20)."""


class UnsupportedError(Exception):
    """MOA_ERR_UNSUPPORTED: a valid request this build / device cannot serve."""


class DeviceError(RunError):
    """MOA_ERR_DEVICE -- CUDA failure."""


class ProviderError(Exception):
    """MOA_ERR_PROVIDER_* -- the reference's ProviderError (errors.hpp:24-33); kind is
    "transport", "missing_credentials" or "bad_response"."""

    def __init__(self, msg, kind):
        super().__init__(msg)
        self.kind = kind


_PROVIDER_KINDS = {6: "transport", 7: "missing_credentials", 8: "bad_response"}
EMBED_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int32), C.c_int, C.c_int, C.POINTER(C.c_double))


class ModelSpec(C.Structure):
    _fields_ = [("tag", C.c_char * 32), ("d", C.c_int), ("n_layers", C.c_int), ("n_heads", C.c_int),
                ("n_kv_heads", C.c_int), ("head_dim", C.c_int), ("ffn", C.c_int), ("vocab", C.c_int),
                ("rope_theta", C.c_double), ("norm_eps", C.c_double), ("lm_gain", C.c_double),
                ("seed", C.c_uint64), ("max_agents", C.c_int)]


class EngineOpts(C.Structure):
    _fields_ = [("max_ctx", C.c_int), ("max_out", C.c_int), ("max_rows", C.c_int), ("device", C.c_int),
                ("keep_logits", C.c_int), ("gemv_only", C.c_int)]


class Event(C.Structure):
    _fields_ = [("kind", C.c_int), ("tick", C.c_int), ("layer", C.c_int), ("position", C.c_int),
                ("a", C.c_int), ("b", C.c_int)]


_P = C.POINTER


class RunConfigC(C.Structure):
    _fields_ = [("topo_kind", C.c_int), ("n_layers", C.c_int), ("widths", _P(C.c_int)),
                ("cluster_sizes", _P(C.c_int)), ("model_cycle", _P(C.c_int)), ("cycle_len", _P(C.c_int)),
                ("out_lo", _P(C.c_int)), ("out_hi", _P(C.c_int)), ("mode", C.c_int), ("early_exit", C.c_int),
                ("exit_scope", C.c_int), ("tau", C.c_double), ("include_diagonal", C.c_int),
                ("use_force_q", C.c_int), ("force_q", C.c_double), ("chunk_size", C.c_int),
                ("seed", C.c_uint64), ("query_tokens", C.c_int), ("leaf_prefix_tokens", C.c_int),
                ("agg_prefix_tokens", C.c_int), ("separator_tokens", C.c_int), ("suffix_tokens", C.c_int),
                ("hidden", C.c_int), ("provider_seed", C.c_uint64), ("embed_model", C.c_int),
                ("embed_fn", EMBED_FN), ("embed_user", C.c_void_p),
                ("out_values", _P(C.c_int)), ("out_values_len", _P(C.c_int))]


class RunSummary(C.Structure):
    _fields_ = [("ticks", C.c_int), ("n_agents", C.c_int), ("n_evals", C.c_int), ("forwards", C.c_int),
                ("tokens", C.c_longlong), ("decoded_tokens", C.c_longlong), ("rows", C.c_longlong),
                ("e2e_ms", C.c_double), ("wall_ms", C.c_double), ("weight_bytes", C.c_double),
                ("host_ms", C.c_double), ("host_wait_ms", C.c_double)]


class AgentRecordC(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("layer", "position", "model", "invoked", "pruned", "empty_input",
                                       "prompt_tokens", "output_tokens", "prefill_only_calls",
                                       "recomputed_tokens", "reclaimed_tokens", "decode_start", "decode_end",
                                       "complete", "precursor_ready")]


class EvalRecordC(C.Structure):
    _fields_ = ([(n, C.c_int) for n in ("tick", "group", "eval_index", "layer", "position", "evaluated", "exited",
                                        "n_pruned", "outputs")]
                + [(n, C.c_double) for n in ("q", "draw", "c", "c_bar", "weight_sum", "weighted", "calibrated")]
                + [("pruned_layer", C.c_int * 16), ("pruned_position", C.c_int * 16)])


class PrefillSpan(C.Structure):
    _fields_ = [("start", C.c_double), ("end", C.c_double), ("wasted", C.c_int)]


class TraceAgent(C.Structure):
    _fields_ = [("layer", C.c_int), ("position", C.c_int), ("model", C.c_int), ("invoked", C.c_int),
                ("pruned", C.c_int), ("prefill_only_calls", C.c_int), ("recomputed_tokens", C.c_int),
                ("complete_t", C.c_double), ("n_prefill", C.c_int), ("prefill", C.POINTER(PrefillSpan))]


class TraceView(C.Structure):
    _fields_ = [("e2e_latency", C.c_double), ("ee_latency_total", C.c_double), ("n_agents", C.c_int),
                ("agents", C.POINTER(TraceAgent))]


SUMMARY_MAX_MODELS = 16


class Summary(C.Structure):
    _fields_ = [("samples", C.c_int), ("mean_e2e", C.c_double), ("p50_e2e", C.c_double), ("p95_e2e", C.c_double),
                ("mean_ee_share", C.c_double), ("mean_prefill_only_calls", C.c_double),
                ("mean_recomputed_tokens", C.c_double), ("prefill_share", C.c_double), ("n_models", C.c_int),
                ("instances", C.c_int * SUMMARY_MAX_MODELS), ("invoked", C.c_int * SUMMARY_MAX_MODELS),
                ("pruned", C.c_int * SUMMARY_MAX_MODELS), ("activation", C.c_double * SUMMARY_MAX_MODELS)]

    def to_dict(self, model_tags=None):
        """RunSummary::to_json field names (orchestrator.cpp:383-402); activation keyed by tag."""
        act = {}
        for m in range(self.n_models):
            if self.instances[m] == 0:
                continue
            tag = model_tags[m] if model_tags else str(m)
            act[tag] = dict(instances=self.instances[m], invoked=self.invoked[m], pruned=self.pruned[m],
                            activation=self.activation[m])
        return dict(samples=self.samples, mean_e2e=self.mean_e2e, p50_e2e=self.p50_e2e, p95_e2e=self.p95_e2e,
                    mean_ee_latency_share=self.mean_ee_share, mean_prefill_only_calls=self.mean_prefill_only_calls,
                    mean_recomputed_tokens=self.mean_recomputed_tokens,
                    critical_path_prefill_share=self.prefill_share, activation=act)


_lib = None

_SIGS = {
    "moa_last_error": ([], C.c_char_p),
    "moa_version": ([], C.c_char_p),
    "moa_device_count": ([_P(C.c_int)], C.c_int),
    "moa_engine_create": ([_P(ModelSpec), C.c_int, _P(EngineOpts), _P(C.c_void_p)], C.c_int),
    "moa_engine_destroy": ([C.c_void_p], C.c_int),
    "moa_engine_reset": ([C.c_void_p], C.c_int),
    "moa_nccl_unique_id": ([_P(C.c_uint8)], C.c_int),
    "moa_engine_attach_comm": ([C.c_void_p, _P(C.c_uint8), C.c_int, C.c_int], C.c_int),
    "moa_loopback_create": ([C.c_int, _P(C.c_void_p)], C.c_int),
    "moa_loopback_destroy": ([C.c_void_p], C.c_int),
    "moa_engine_attach_loopback": ([C.c_void_p, C.c_void_p, C.c_int], C.c_int),
    "moa_placement": ([C.c_int, C.c_int, _P(C.c_int), _P(C.c_int), C.c_int, _P(C.c_int)], C.c_int),
    "moa_k_noop": ([C.c_size_t, C.c_int, C.c_size_t], C.c_int),
    "moa_k_chain_stamp": ([C.c_size_t], C.c_int),
    "moa_engine_probe": ([C.c_void_p, C.c_int], C.c_int),
    "moa_engine_probe_stats": ([C.c_void_p, C.c_int, _P(C.c_int), _P(C.c_double), _P(C.c_double), _P(C.c_double)],
                               C.c_int),
    "moa_add_agent": ([C.c_void_p, C.c_int, C.c_int, C.c_int], C.c_int),
    "moa_prefill_only": ([C.c_void_p, C.c_int, C.c_int, C.c_int, _P(C.c_int32), C.c_int], C.c_int),
    "moa_generate": ([C.c_void_p, C.c_int, C.c_int, _P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int], C.c_int),
    "moa_cancel": ([C.c_void_p, C.c_int, C.c_int], C.c_int),
    "moa_reclaim": ([C.c_void_p, C.c_int, C.c_int, C.c_int], C.c_int),
    "moa_step": ([C.c_void_p, _P(Event), C.c_int, _P(C.c_int), _P(C.c_int)], C.c_int),
    "moa_busy": ([C.c_void_p, _P(C.c_int)], C.c_int),
    "moa_read_output": ([C.c_void_p, C.c_int, C.c_int, C.c_int, _P(C.c_int32), _P(C.c_float), _P(C.c_float)],
                        C.c_int),
    "moa_read_logits": ([C.c_void_p, C.c_int, C.c_int, C.c_int, _P(C.c_float), C.c_int], C.c_int),
    "moa_agent_state": ([C.c_void_p, C.c_int, C.c_int] + [_P(C.c_int)] * 4, C.c_int),
    "moa_engine_trace": ([C.c_void_p, C.c_int], C.c_int),
    "moa_read_residual": ([C.c_void_p, C.c_int, C.c_int, _P(C.c_float), C.c_longlong], C.c_int),
    "moa_engine_mark_start": ([C.c_void_p], C.c_int),
    "moa_engine_tick": ([C.c_void_p, _P(C.c_int)], C.c_int),
    "moa_tick_seconds": ([C.c_void_p, C.c_int, _P(C.c_double)], C.c_int),
    "moa_agent_record_get": ([C.c_void_p, C.c_int, C.c_int, _P(AgentRecordC)], C.c_int),
    "moa_query_trace": ([C.c_void_p, C.c_char_p, C.c_longlong, _P(C.c_longlong)], C.c_int),
    "moa_query_ticks": ([C.c_void_p, _P(C.c_double), C.c_int, _P(C.c_int)], C.c_int),
    "moa_run_batch": ([C.c_void_p, C.c_void_p, _P(C.c_int), C.c_int, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "moa_run_query": ([C.c_void_p, _P(RunConfigC), C.c_int, C.c_int, _P(RunSummary), _P(C.c_void_p)], C.c_int),
    "moa_query_agent": ([C.c_void_p, C.c_int, _P(AgentRecordC)], C.c_int),
    "moa_query_tokens": ([C.c_void_p, C.c_int, C.c_int, _P(C.c_int32), C.c_int, _P(C.c_int)], C.c_int),
    "moa_query_logprobs": ([C.c_void_p, C.c_int, _P(C.c_float), _P(C.c_float), C.c_int, _P(C.c_int)], C.c_int),
    "moa_query_eval": ([C.c_void_p, C.c_int, _P(EvalRecordC), _P(C.c_double), C.c_int], C.c_int),
    "moa_query_free": ([C.c_void_p], C.c_int),
    "moa_summarize": ([C.c_int, C.c_int, _P(C.c_int), _P(C.c_int), _P(TraceView), C.c_int, _P(Summary)], C.c_int),
    "moa_percentile": ([_P(C.c_double), C.c_int, C.c_double, _P(C.c_double)], C.c_int),
    "moa_run_repetitions": ([C.c_void_p, _P(RunConfigC), C.c_int, _P(Summary), C.c_void_p], C.c_int),
    "moa_query_trace_view": ([C.c_void_p, _P(TraceView), _P(TraceAgent), C.c_int, _P(PrefillSpan), C.c_int,
                              _P(C.c_int), _P(C.c_int)], C.c_int),
    "moa_mock_embed": ([_P(C.c_int32), C.c_int, C.c_int, C.c_uint64, _P(C.c_double), C.c_int], C.c_int),
    "moa_metricq_run": ([_P(C.c_int32), _P(C.c_float), _P(C.c_int), C.c_int, C.c_int, C.c_uint64, C.c_double,
                         C.c_int, C.c_uint64, C.c_char_p, _P(C.c_double), _P(C.c_double), _P(C.c_int),
                         _P(C.c_double), C.c_int], C.c_int),
    "moa_mq_group_create": ([C.c_int, C.c_uint64, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _P(C.c_void_p)],
                            C.c_int),
    "moa_mq_group_add_completion": ([C.c_void_p, _P(C.c_int32), _P(C.c_double), C.c_int, C.c_void_p,
                                     _P(C.c_double), C.c_int], C.c_int),
    "moa_mq_group_add_embedded": ([C.c_void_p, _P(C.c_double), _P(C.c_double), C.c_int, C.c_void_p,
                                   _P(C.c_double), C.c_int], C.c_int),
    "moa_mq_group_completions": ([C.c_void_p, _P(C.c_int)], C.c_int),
    "moa_mq_group_free": ([C.c_void_p], C.c_int),
    "moa_rng_derive": ([C.c_uint64, C.c_char_p, _P(C.c_uint64)], C.c_int),
    "moa_decide_exit": ([C.c_double, _P(C.c_uint64), _P(C.c_double), _P(C.c_int)], C.c_int),
    "moa_topology": ([C.c_int, C.c_int, _P(C.c_int), _P(C.c_int), _P(C.c_int), _P(C.c_int), C.c_int], C.c_int),
    "moa_slotplan_create": ([C.c_int, C.c_int, _P(C.c_int32), C.c_int, _P(C.c_int), _P(C.c_int), _P(C.c_int32),
                             _P(C.c_int), C.c_int, _P(C.c_int32), C.c_int, C.c_int, _P(C.c_void_p)], C.c_int),
    "moa_slotplan_event": ([C.c_void_p, C.c_int, C.c_int, C.c_int, _P(C.c_int32), C.c_int, _P(C.c_int32), C.c_int,
                            _P(C.c_int)], C.c_int),
    "moa_slotplan_free": ([C.c_void_p], C.c_int),
    "moa_k_attention": ([C.c_size_t, C.c_size_t, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_size_t,
                         C.c_size_t, C.c_longlong, C.c_int, C.c_size_t, C.c_int, C.c_size_t, C.c_int], C.c_int),
    "moa_k_gemv": ([C.c_size_t, C.c_size_t, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_size_t, C.c_size_t], C.c_int),
    "moa_k_gemm_tc": ([C.c_size_t, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_size_t, C.c_size_t], C.c_int),
    "moa_k_gemv_tc": ([C.c_size_t, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_size_t, C.c_size_t], C.c_int),
    "moa_k_init_uniform": ([C.c_size_t, C.c_longlong, C.c_longlong, C.c_uint64, C.c_float, C.c_int, C.c_int,
                            C.c_size_t], C.c_int),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load libmoa_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2512_18126_b200.build`")
        L = C.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        _lib = L
    return _lib


def check(rc: int):
    if rc == MOA_OK:
        return
    msg = lib().moa_last_error().decode(errors="replace")
    if rc == MOA_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == MOA_ERR_DEVICE:
        raise DeviceError(msg)
    if rc in _PROVIDER_KINDS:
        raise ProviderError(msg, _PROVIDER_KINDS[rc])
    if rc == MOA_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    raise RunError(msg)


def _ints(v):
    v = [int(x) for x in v]
    return (C.c_int32 * max(1, len(v)))(*v), len(v)


SHAPES = {
    "tiny": dict(d=256, n_layers=4, n_heads=4, n_kv_heads=4, head_dim=64, ffn=1024),
    "1b": dict(d=2048, n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, ffn=8192),
    "8b": dict(d=4096, n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336),
}


def model_spec(tag: str, shape: str, seed: int = 0, max_agents: int = 16, vocab: int = 50000,
               lm_gain: float = 4.0, **over) -> ModelSpec:
    """`over` overrides shape fields (e.g. n_layers=2: the shape's first layers, same weights)."""
    s = {**SHAPES[shape], **over}
    return ModelSpec(tag=tag.encode()[:31], vocab=vocab, rope_theta=10000.0, norm_eps=1e-5, lm_gain=lm_gain,
                     seed=seed, max_agents=max_agents, **s)


class Engine:
    """Owns one moa_engine (one GPU)."""

    def __init__(self, models, max_ctx=1024, max_out=1024, max_rows=16384, device=0, keep_logits=False,
                 gemv_only=False):
        self.models = list(models)
        arr = (ModelSpec * len(self.models))(*self.models)
        opts = EngineOpts(max_ctx, max_out, max_rows, device, int(keep_logits), int(gemv_only))
        h = C.c_void_p()
        check(lib().moa_engine_create(arr, len(self.models), C.byref(opts), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            check(lib().moa_engine_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- SimWorld protocol ---
    def add_agent(self, a, model):
        check(lib().moa_add_agent(self.h, a[0], a[1], model))

    def prefill_only(self, a, start, tokens):
        buf, n = _ints(tokens)
        check(lib().moa_prefill_only(self.h, a[0], a[1], start, buf, n))

    def generate(self, a, prompt, max_new, apc_chunk, prefill_chunk=0):
        buf, n = _ints(prompt)
        check(lib().moa_generate(self.h, a[0], a[1], buf, n, max_new, apc_chunk, prefill_chunk))

    def cancel(self, a):
        check(lib().moa_cancel(self.h, a[0], a[1]))

    def reclaim(self, a, keep):
        check(lib().moa_reclaim(self.h, a[0], a[1], keep))

    def step(self):
        ev = (Event * 256)()
        n, busy = C.c_int(), C.c_int()
        check(lib().moa_step(self.h, ev, 256, C.byref(n), C.byref(busy)))
        out = [(EVENT_KINDS[e.kind], e.tick, (e.layer, e.position), e.a, e.b) for e in ev[: min(n.value, 256)]]
        return out, bool(busy.value)

    def busy(self):
        b = C.c_int()
        check(lib().moa_busy(self.h, C.byref(b)))
        return bool(b.value)

    def read_output(self, a, n):
        tok, lp, ent = (C.c_int32 * max(n, 1))(), (C.c_float * max(n, 1))(), (C.c_float * max(n, 1))()
        check(lib().moa_read_output(self.h, a[0], a[1], n, tok, lp, ent))
        return list(tok[:n]), list(lp[:n]), list(ent[:n])

    def read_logits(self, a, k):
        vocab = self.models[self.record(a)["model"]].vocab
        buf = (C.c_float * vocab)()
        check(lib().moa_read_logits(self.h, a[0], a[1], k, buf, vocab))
        import numpy as np
        return np.ctypeslib.as_array(buf).copy()

    def read_residual(self, model: int, rows: int):
        """fp32 residual rows [rows][d] of the model's last forward (test hook)."""
        import numpy as np
        d = self.models[model].d
        buf = np.zeros(rows * d, dtype=np.float32)
        check(lib().moa_read_residual(self.h, model, rows, buf.ctypes.data_as(_P(C.c_float)), buf.size))
        return buf.reshape(rows, d)

    def state(self, a):
        v = [C.c_int() for _ in range(4)]
        check(lib().moa_agent_state(self.h, a[0], a[1], *[C.byref(x) for x in v]))
        return dict(zip(("scheduled", "decoded", "finished", "cancelled"), (x.value for x in v)))

    def reset(self):
        check(lib().moa_engine_reset(self.h))

    def mark_start(self):
        """Time zero of tick_seconds (engine stream)."""
        check(lib().moa_engine_mark_start(self.h))

    def tick(self) -> int:
        """Ticks run so far (the index of the next tick)."""
        v = C.c_int()
        check(lib().moa_engine_tick(self.h, C.byref(v)))
        return v.value

    def tick_seconds(self, tick: int) -> float:
        """Device seconds from mark_start to the end of `tick` (needs trace(True) while it ran)."""
        v = C.c_double()
        check(lib().moa_tick_seconds(self.h, tick, C.byref(v)))
        return v.value

    def record(self, a) -> dict:
        r = AgentRecordC()
        check(lib().moa_agent_record_get(self.h, a[0], a[1], C.byref(r)))
        return {k: getattr(r, k) for k, _ in AgentRecordC._fields_}

    def attach_comm(self, nccl_id: bytes, rank: int, world: int):
        """Join a tree-partitioned serving group (call before the first request)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        check(lib().moa_engine_attach_comm(self.h, buf, rank, world))

    def attach_loopback(self, hub: "LoopbackHub", rank: int):
        """Join an in-process partitioned group (one thread per engine)."""
        check(lib().moa_engine_attach_loopback(self.h, hub.h, rank))
        self._hub = hub  # keep the hub alive as long as the engine

    # include/moa_b200.h moa_engine_probe_stats: decode-regime kinds, then prefill-regime kinds
    PROBE_KINDS = ("embed", "qkv", "attn_decode", "o_proj", "gate_up", "down", "lm_head", "qkv_attn",
                   "attn_prefill", "pf_qkv", "pf_o_proj", "pf_gate_up", "pf_down")
    PREFILL_KINDS = ("attn_prefill", "pf_qkv", "pf_o_proj", "pf_gate_up", "pf_down")

    def probe(self, enable: bool):
        check(lib().moa_engine_probe(self.h, int(enable)))

    def probe_stats(self):
        out = {}
        for k, name in enumerate(self.PROBE_KINDS):
            n, ms, b, f = C.c_int(), C.c_double(), C.c_double(), C.c_double()
            check(lib().moa_engine_probe_stats(self.h, k, C.byref(n), C.byref(ms), C.byref(b), C.byref(f)))
            out[name] = {"launches": n.value, "ms": ms.value, "bytes": b.value, "flops": f.value}
        return out

    # --- run_query ---
    def run_batch(self, cfg: "QueryConfig", samples, resolve=True, detail=True):
        """Concurrent requests (continuous batching); one result dict per sample."""
        n = len(samples)
        arr = (C.c_int * n)(*samples)
        sums = (RunSummary * n)()
        qs = (C.c_void_p * n)()
        check(lib().moa_run_batch(self.h, C.byref(cfg.c), arr, n, int(resolve), sums, qs if detail else None))
        out = []
        for i in range(n):
            res = {k: getattr(sums[i], k) for k, _ in RunSummary._fields_}
            if detail:
                try:
                    res.update(_query_detail(C.c_void_p(qs[i]), sums[i], resolve))
                finally:
                    lib().moa_query_free(C.c_void_p(qs[i]))
            out.append(res)
        return out

    def run_repetitions(self, cfg: "QueryConfig", repetitions: int):
        """run_repetitions + summarize (orchestrator.cpp:297-382) on the GPU: samples
        0..repetitions-1, device seconds.  Returns (summary dict, per-sample summaries)."""
        out = Summary()
        per = (RunSummary * repetitions)()
        check(lib().moa_run_repetitions(self.h, C.byref(cfg.c), int(repetitions), C.byref(out), per))
        rows = [{k: getattr(per[i], k) for k, _ in RunSummary._fields_} for i in range(repetitions)]
        return out.to_dict(cfg.model_tags), rows

    def trace(self, enable: bool = True):
        """Record per-tick device times so run_query(..., trace=True) returns a RunTrace JSONL."""
        check(lib().moa_engine_trace(self.h, int(enable)))

    def run_query(self, cfg: "QueryConfig", sample=0, resolve=True, detail=True, trace=False):
        s = RunSummary()
        q = C.c_void_p()
        check(lib().moa_run_query(self.h, C.byref(cfg.c), sample, int(resolve), C.byref(s),
                                  C.byref(q) if (detail or trace) else None))
        res = {k: getattr(s, k) for k, _ in RunSummary._fields_}
        if detail or trace:
            try:
                if detail:
                    res.update(_query_detail(q, s, resolve))
                if trace:
                    n = C.c_longlong()
                    check(lib().moa_query_trace(q, None, 0, C.byref(n)))
                    buf = C.create_string_buffer(n.value + 1)
                    check(lib().moa_query_trace(q, buf, n.value + 1, C.byref(n)))
                    res["trace"] = buf.value.decode()
                    nt = C.c_int()
                    check(lib().moa_query_ticks(q, None, 0, C.byref(nt)))
                    tb = (C.c_double * max(1, nt.value))()
                    check(lib().moa_query_ticks(q, tb, nt.value, C.byref(nt)))
                    res["tick_ms"] = list(tb[: nt.value])
                    res["trace_view"] = _trace_view(q, cfg.model_tags)
            finally:
                lib().moa_query_free(q)
        return res


def _trace_view(q, model_tags):
    """moa_query_trace_view as the dict capi.summarize takes (device seconds)."""
    na, ns = C.c_int(), C.c_int()
    check(lib().moa_query_trace_view(q, None, None, 0, None, 0, C.byref(na), C.byref(ns)))
    ags, sps, view = (TraceAgent * max(1, na.value))(), (PrefillSpan * max(1, ns.value))(), TraceView()
    check(lib().moa_query_trace_view(q, C.byref(view), ags, na.value, sps, ns.value, C.byref(na), C.byref(ns)))
    agents = []
    for i in range(na.value):
        a = ags[i]
        agents.append(dict(layer=a.layer, position=a.position, model_tag=model_tags[a.model], invoked=bool(a.invoked),
                           pruned=bool(a.pruned), prefill_only_calls=a.prefill_only_calls,
                           recomputed_tokens=a.recomputed_tokens, complete_t=a.complete_t,
                           prefill=[(a.prefill[j].start, a.prefill[j].end, bool(a.prefill[j].wasted))
                                    for j in range(a.n_prefill)]))
    return dict(e2e_latency=view.e2e_latency, ee_latency_total=view.ee_latency_total, agents=agents)


def _query_detail(q, s, resolve):
    agents, evals = {}, []
    for i in range(s.n_agents):
        r = AgentRecordC()
        check(lib().moa_query_agent(q, i, C.byref(r)))
        d = {k: getattr(r, k) for k, _ in AgentRecordC._fields_}
        if resolve:
            for which, key in ((0, "prompt"), (1, "output")):
                n = C.c_int()
                check(lib().moa_query_tokens(q, i, which, None, 0, C.byref(n)))
                buf = (C.c_int32 * max(1, n.value))()
                check(lib().moa_query_tokens(q, i, which, buf, n.value, C.byref(n)))
                d[key] = list(buf[: n.value])
            n = C.c_int()
            cap = max(1, len(d["output"]))
            lp, ent = (C.c_float * cap)(), (C.c_float * cap)()
            check(lib().moa_query_logprobs(q, i, lp, ent, cap, C.byref(n)))
            d["logprobs"], d["entropy"] = list(lp[: n.value]), list(ent[: n.value])
        agents[f"{r.layer}:{r.position}"] = d
    for i in range(s.n_evals):
        e = EvalRecordC()
        row = (C.c_double * 64)()
        check(lib().moa_query_eval(q, i, C.byref(e), row, 64))
        d = {k: getattr(e, k) for k, _ in EvalRecordC._fields_ if not k.startswith("pruned_")}
        d["completed"] = f"{e.layer}:{e.position}"
        d["pruned"] = [f"{e.pruned_layer[k]}:{e.pruned_position[k]}" for k in range(e.n_pruned)]
        d["sim_row"] = list(row[: e.outputs])
        evals.append(d)
    return dict(agents=agents, metricq=evals)


class QueryConfig:
    """moa_run_config built from a plain config dict (configs.py)."""

    def __init__(self, cfg: dict, model_index: dict, embed=None):
        """embed: optional EmbeddingProvider (embedding.hpp:38-44), a callable
        tokens -> array [n][cfg["hidden"]] (fp64) used by the early-exit gate
        instead of the mock; it may raise ProviderError."""
        t = cfg["topology"]
        widths = list(t["widths"])
        L = len(widths)
        self._keep = []
        self.model_tags = [k for k, _ in sorted(model_index.items(), key=lambda kv: kv[1])]

        def arr(v, ty=C.c_int):
            a = (ty * max(1, len(v)))(*v)
            self._keep.append(a)
            return C.cast(a, _P(ty))

        if t["kind"] == "all_to_all":
            kind, cs = 1, None
        else:
            kind = 0
            if "cluster_sizes" in t:
                sizes = [s for layer in t["cluster_sizes"] for s in layer]
            else:
                sizes = [b for l, b in enumerate(t["branching"]) for _ in range(widths[l + 1])]
            cs = arr(sizes)
        cyc, clen, lo, hi, vals, vlen = [], [], [], [], [], []
        for l in range(L):
            c = cfg["assign"][min(l, len(cfg["assign"]) - 1)]
            cyc += [model_index[x] for x in c]
            clen.append(len(c))
            ol = cfg["out_len"][min(l, len(cfg["out_len"]) - 1)]
            if isinstance(ol, dict):  # OutputLenDist::Empirical
                a = b = 0
                vals += list(ol["values"])
                vlen.append(len(ol["values"]))
            else:
                a, b = (ol, ol) if isinstance(ol, int) else tuple(ol)
                vlen.append(0)
            lo.append(a)
            hi.append(b)
        fq = cfg.get("force_q")
        self.c = RunConfigC(
            topo_kind=kind, n_layers=L, widths=arr(widths), cluster_sizes=cs, model_cycle=arr(cyc),
            cycle_len=arr(clen), out_lo=arr(lo), out_hi=arr(hi), mode=MODES[cfg["mode"]],
            early_exit=int(cfg["early_exit"]), exit_scope=0 if cfg.get("exit_scope", "cluster") == "cluster" else 1,
            tau=cfg.get("tau", 0.7), include_diagonal=int(cfg.get("include_diagonal", True)),
            use_force_q=int(fq is not None), force_q=fq or 0.0, chunk_size=cfg["chunk_size"], seed=cfg["seed"],
            query_tokens=cfg["query_tokens"], leaf_prefix_tokens=cfg["leaf_prefix_tokens"],
            agg_prefix_tokens=cfg["agg_prefix_tokens"], separator_tokens=cfg["separator_tokens"],
            suffix_tokens=cfg["suffix_tokens"], hidden=cfg.get("hidden", 64),
            provider_seed=cfg.get("provider_seed", 0),
            embed_model=model_index[cfg["embed_model"]] if cfg.get("provider", "mock") == "hidden" else -1,
            out_values=arr(vals) if vals else None, out_values_len=arr(vlen))
        if embed is not None:
            import numpy as np
            codes = {v: k for k, v in _PROVIDER_KINDS.items()}

            def _cb(user, toks, n, hidden, out):
                try:
                    e = np.ascontiguousarray(np.asarray(embed([toks[i] for i in range(n)]), dtype=np.float64))
                    if e.shape != (n, hidden):
                        return MOA_ERR_PROVIDER_BAD_RESPONSE
                    C.memmove(out, e.ctypes.data, e.nbytes)
                    return MOA_OK
                except ProviderError as ex:
                    return codes.get(ex.kind, MOA_ERR_PROVIDER_BAD_RESPONSE)
                except Exception:
                    return MOA_ERR_PROVIDER_BAD_RESPONSE

            self._embed_cb = EMBED_FN(_cb)  # kept alive with the config
            self.c.embed_fn = self._embed_cb


def engine_for(cfg: dict, device=0, keep_logits=False, max_ctx=None, max_rows=16384, gemv_only=False, concurrency=1,
               embed=None):
    """Engine holding every model the config names, sized for its agents
    (times `concurrency` requests served at once by run_batch)."""
    from collections import Counter
    counts = Counter()
    t = cfg["topology"]
    for l, w in enumerate(t["widths"]):
        for p in range(w):
            counts[_configs.agent_tag(cfg, l + 1, p)] += 1
    if cfg.get("provider", "mock") == "hidden":  # the hidden-state provider reserves one KV slot of its model
        counts[cfg["embed_model"]] += 1
    tags = list(cfg["models"])
    specs = [model_spec(tag, cfg["models"][tag]["shape"], cfg["models"][tag].get("seed", 0),
                        max_agents=max(1, counts[tag] * concurrency),
                        **{k: v for k, v in cfg["models"][tag].items() if k not in ("shape", "seed")})
             for tag in tags]
    out_max = max(x if isinstance(x, int) else max(x["values"]) if isinstance(x, dict) else x[1]
                  for x in cfg["out_len"])
    if max_ctx is None:
        prompt_max = max(cfg["query_tokens"] + cfg["leaf_prefix_tokens"],
                         cfg["agg_prefix_tokens"] + cfg["suffix_tokens"]
                         + max(t["widths"]) * (out_max + cfg["separator_tokens"]))
        max_ctx = ((prompt_max + out_max + 255) // 256) * 256
    eng = Engine(specs, max_ctx=max_ctx, max_out=out_max, max_rows=max_rows, device=device, keep_logits=keep_logits,
                 gemv_only=gemv_only)
    return eng, QueryConfig(cfg, {t: i for i, t in enumerate(tags)}, embed=embed)


class Quality(C.Structure):
    _fields_ = [("outputs", C.c_int)] + [(n, C.c_double) for n in ("c", "c_bar", "weight_sum", "weighted",
                                                                    "calibrated", "q", "tau")]


class MetricQGroup:
    """One exit group's incremental evaluator on the GPU (moa_mq_group_*,
    the reference's MetricQEvaluator, metricq.hpp:102-122)."""

    def __init__(self, hidden: int, provider_seed: int = 0, tau: float = 0.7, include_diagonal: bool = True,
                 max_members: int = 16, max_tokens: int = 4096, device: int = 0):
        h = C.c_void_p()
        check(lib().moa_mq_group_create(hidden, provider_seed, tau, int(include_diagonal), max_members, max_tokens,
                                        device, C.byref(h)))
        self.h, self.hidden, self.max_members = h, hidden, max_members

    def _result(self, q, sim):
        n = q.outputs
        import numpy as np
        d = {k: getattr(q, k) for k, _ in Quality._fields_}
        d["sim"] = np.array(sim[: n * n]).reshape(n, n)
        return d

    def add_completion(self, tokens, logprobs):
        """MockProvider embeddings of `tokens` (device)."""
        n = len(tokens)
        q, sim = Quality(), (C.c_double * (self.max_members ** 2))()
        check(lib().moa_mq_group_add_completion(self.h, (C.c_int32 * n)(*tokens), (C.c_double * n)(*logprobs), n,
                                                C.byref(q), sim, self.max_members ** 2))
        return self._result(q, sim)

    def add_embedded(self, emb, logprobs):
        """Rows from any EmbeddingProvider: emb [n][hidden] fp64."""
        import numpy as np
        e = np.ascontiguousarray(emb, dtype=np.float64)
        n = e.shape[0]
        q, sim = Quality(), (C.c_double * (self.max_members ** 2))()
        check(lib().moa_mq_group_add_embedded(self.h, e.ctypes.data_as(_P(C.c_double)), (C.c_double * n)(*logprobs),
                                              n, C.byref(q), sim, self.max_members ** 2))
        return self._result(q, sim)

    def completions(self) -> int:
        n = C.c_int()
        check(lib().moa_mq_group_completions(self.h, C.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            lib().moa_mq_group_free(self.h)
            self.h = None

    __del__ = close


def rng_derive(master: int, label: str) -> int:
    s = C.c_uint64()
    check(lib().moa_rng_derive(master, label.encode(), C.byref(s)))
    return s.value


def decide_exit(q: float, state: int):
    """(draw, exited, next state) -- decide_exit (metricq.cpp:125-131) on an RngStream state."""
    s, d, e = C.c_uint64(state), C.c_double(), C.c_int()
    check(lib().moa_decide_exit(q, C.byref(s), C.byref(d), C.byref(e)))
    return d.value, bool(e.value), s.value


def device_count() -> int:
    n = C.c_int()
    check(lib().moa_device_count(C.byref(n)))
    return n.value


if os.environ.get("MOA_B200_EAGER_LOAD"):
    lib()


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().moa_nccl_unique_id(buf))
    return bytes(buf)


class LoopbackHub:
    """In-process stand-in for the NCCL group (see include/moa_b200.h)."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib().moa_loopback_create(world, C.byref(h)))
        self.h, self.world = h, world

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            lib().moa_loopback_destroy(self.h)
            self.h = None


def placement(topology: dict, world: int) -> dict:
    """Owning rank per agent ("l:p") for tree-partitioned serving."""
    widths = list(topology["widths"])
    kind = 1 if topology["kind"] == "all_to_all" else 0
    cs = None
    if kind == 0:
        if "cluster_sizes" in topology:
            sizes = [s for layer in topology["cluster_sizes"] for s in layer]
        else:
            sizes = [b for l, b in enumerate(topology["branching"]) for _ in range(widths[l + 1])]
        cs = (C.c_int * max(1, len(sizes)))(*sizes)
    w = (C.c_int * len(widths))(*widths)
    out = (C.c_int * sum(widths))()
    check(lib().moa_placement(kind, len(widths), w, cs, world, out))
    names = [f"{l + 1}:{p}" for l, n in enumerate(widths) for p in range(n)]
    return dict(zip(names, list(out)))


class SlotPlan:
    """Incremental slot filling of one consumer (router.cpp:38-184) over the
    C-ABI moa_slotplan_*: each event returns the engine actions it triggers,
    as dicts {"kind": "prefill_only"|"generate"|"reclaim", "start", "tokens"}."""

    _OPS = {"start": 0, "chunk": 1, "done": 2, "cancelled": 3}
    _KINDS = {0: "prefill_only", 1: "generate", 2: "reclaim"}

    def __init__(self, self_id, prefix, slots, suffix, incremental=True):
        """slots: [(producer (layer, position), separator tokens), ...] in slot order."""
        sl = (C.c_int * max(1, len(slots)))(*[int(p[0]) for p, _ in slots])
        sp = (C.c_int * max(1, len(slots)))(*[int(p[1]) for p, _ in slots])
        seps = [int(t) for _, sep in slots for t in sep]
        st = (C.c_int32 * max(1, len(seps)))(*seps)
        sn = (C.c_int * max(1, len(slots)))(*[len(sep) for _, sep in slots])
        pre, npre = _ints(prefix)
        suf, nsuf = _ints(suffix)
        h = C.c_void_p()
        check(lib().moa_slotplan_create(int(self_id[0]), int(self_id[1]), pre, npre, sl, sp, st, sn, len(slots), suf,
                                        nsuf, int(bool(incremental)), C.byref(h)))
        self.h = h
        self.self_id = (int(self_id[0]), int(self_id[1]))

    def _event(self, op, producer=(0, 0), tokens=()):
        tb, n = _ints(tokens)
        cap = 1 << 16
        buf = (C.c_int32 * cap)()
        nw = C.c_int()
        check(lib().moa_slotplan_event(self.h, self._OPS[op], int(producer[0]), int(producer[1]), tb, n, buf, cap,
                                       C.byref(nw)))
        out, i = [], 0
        while i < nw.value:
            k, s, m = buf[i], buf[i + 1], buf[i + 2]
            out.append({"kind": self._KINDS[k], "start": s, "tokens": list(buf[i + 3:i + 3 + m])})
            i += 3 + m
        return out

    def start(self):
        return self._event("start")

    def on_chunk(self, producer, tokens):
        return self._event("chunk", producer, tokens)

    def on_precursor_done(self, producer):
        return self._event("done", producer)

    def on_precursor_cancelled(self, producer):
        return self._event("cancelled", producer)

    def close(self):
        if self.h:
            lib().moa_slotplan_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def summarize(topology: dict, traces, model_index: dict):
    """moa_summarize over traces given as dicts {e2e_latency, ee_latency_total,
    agents: [{layer, position, model_tag, invoked, pruned, prefill_only_calls,
    recomputed_tokens, complete_t, prefill: [(start, end, wasted)]}]}."""
    kind = 1 if topology["kind"] == "all_to_all" else 0
    widths = topology["widths"]
    w = (C.c_int * len(widths))(*widths)
    cs = None
    if kind == 0:
        br = topology.get("branching", [])
        sizes = [br[l] for l in range(len(widths) - 1) for _ in range(widths[l + 1])]
        cs = (C.c_int * max(1, len(sizes)))(*sizes)
    keep, views = [], (TraceView * max(1, len(traces)))()
    for i, t in enumerate(traces):
        ags = (TraceAgent * max(1, len(t["agents"])))()
        for k, a in enumerate(t["agents"]):
            sp = (PrefillSpan * max(1, len(a["prefill"])))(*[PrefillSpan(p[0], p[1], int(p[2])) for p in a["prefill"]])
            keep.append(sp)
            ags[k] = TraceAgent(a["layer"], a["position"], model_index[a["model_tag"]], int(a["invoked"]),
                                int(a["pruned"]), a["prefill_only_calls"], a["recomputed_tokens"], a["complete_t"],
                                len(a["prefill"]), sp)
        keep.append(ags)
        views[i] = TraceView(t["e2e_latency"], t["ee_latency_total"], len(t["agents"]), ags)
    out = Summary()
    check(lib().moa_summarize(kind, len(widths), w, cs, views, len(traces), C.byref(out)))
    tags = {v: k for k, v in model_index.items()}
    return out.to_dict([tags.get(m, str(m)) for m in range(out.n_models)])


def percentile(v, p: float) -> float:
    arr = (C.c_double * max(1, len(v)))(*v)
    out = C.c_double()
    check(lib().moa_percentile(arr, len(v), float(p), C.byref(out)))
    return out.value
