"""Parity helpers (test infrastructure): teacher-forced numerics and
record-and-replay of a GPU request through the oracle orchestration.

Tolerance rationale: activations are rounded to bf16 at the
same points on both sides, but fp32 accumulation order differs, which flips
individual bf16 roundings; the oracle against an fp64-accumulation variant of
itself already differs by up to ~0.08 in the logits (tests/test_oracle_
sensitivity.py).  LOGIT_ATOL is twice the measured self-sensitivity; greedy
ids are compared wherever the oracle's top-1 margin exceeds 2*LOGIT_ATOL.
"""
from __future__ import annotations

import numpy as np

from .model import CpuModel, logit_stats

LOGIT_ATOL = 0.2
# logprob = x_tok - logsumexp(x): its error is at most |d x_tok| + max |d x| <= 2 x LOGIT_ATOL; 0.1 (half a
# logit bound) is the bar, observed max 0.052 on tiny agents and 0.023 on 8B-width ones
LOGPROB_ATOL = 0.1


def teacher_forced(model: CpuModel, prompt, outputs):
    """Logits predicting outputs[k] given prompt + outputs[:k] (one prefill
    over the whole sequence on a fresh KV)."""
    seq = list(prompt) + list(outputs[:-1]) if outputs else list(prompt)
    P, n = len(prompt), len(outputs)
    if n == 0:
        return np.zeros((0, model.spec.vocab), np.float32)
    kv = model.new_kv()
    want = [i >= P - 1 for i in range(len(seq))]
    if P == 0:  # empty prompt: BOS 0 bootstraps (engine contract)
        seq = [0] + list(outputs[:-1])
        want = [True] * len(seq)
    return model.forward([(kv, i, t) for i, t in enumerate(seq)], want)


def check_agent(model: CpuModel, prompt, out_tokens, out_logprobs, logits_atol=LOGIT_ATOL, lp_atol=LOGPROB_ATOL,
                gpu_logits=None):
    """Returns dict(checked, skipped_near_tie, mismatches, max_lp_err).  A
    mismatch is a GPU greedy id that disagrees with a decisive oracle argmax.

    With the GPU's own fp32 logits (keep_logits engines) the bound is the
    measured one, per logit: every logit of token k must be within logits_atol
    of the oracle's, and token k is decisive when the oracle's argmax a beats
    every other id v by more than the two measured errors, L_a - L_v >
    |dL_a| + |dL_v| -- then the GPU argmax provably equals the oracle's.
    Without them the margin must exceed 2 * logits_atol."""
    L = teacher_forced(model, prompt, out_tokens)
    tok, lp, _ = logit_stats(L)
    srt = np.sort(L, axis=-1)
    margin = srt[:, -1] - srt[:, -2]
    n = len(out_tokens)
    bound = np.full(n, logits_atol)
    logit_err = None
    decisive = margin > 2 * bound
    if gpu_logits is not None:
        G = np.asarray(gpu_logits, dtype=np.float32).reshape(L.shape)
        E = np.abs(G - L)
        err_k = E.max(axis=-1) if n else np.zeros(0)
        logit_err = float(err_k.max()) if n else 0.0
        # pairwise bound: with measured per-logit errors e_v, the GPU ranks the
        # oracle's argmax a above every v whenever L_a - L_v > e_a + e_v, so
        # token k is decisive when min_v (L_a - e_a - L_v - e_v) > 0 (and every
        # error is within logits_atol)
        a = L.argmax(axis=-1)
        ea = E[np.arange(n), a]
        la = L[np.arange(n), a]
        slack = (la - ea)[:, None] - (L + E)
        slack[np.arange(n), a] = np.inf
        decisive = (slack.min(axis=-1) > 0) & (err_k <= logits_atol) if n else np.zeros(0, bool)
    mism = [k for k in range(n) if decisive[k] and int(tok[k]) != int(out_tokens[k])]
    # logprob of the GPU's token under the oracle
    z = L - L.max(axis=-1, keepdims=True)
    lse = np.log(np.exp(z).sum(axis=-1))
    lp_gpu_tok = np.array([z[k, out_tokens[k]] - lse[k] for k in range(n)])
    lp_errs = np.abs(lp_gpu_tok - np.asarray(out_logprobs)) if n else np.zeros(0)
    lp_err = float(lp_errs.max()) if n else 0.0
    if logit_err is not None:
        # the GPU's logprob is its own logit minus its own log-sum-exp, so its
        # error against the oracle is at most twice that token's logit error
        lp_ok = logit_err <= logits_atol and bool(np.all(lp_errs <= 2 * err_k + 1e-4))
    else:
        lp_ok = lp_err <= lp_atol
    return dict(checked=int(decisive.sum()), skipped_near_tie=int((~decisive).sum()), mismatches=mism,
                max_lp_err=lp_err, lp_ok=lp_ok, max_logit_err=logit_err)
