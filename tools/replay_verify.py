"""Replay verifier for GPU RunTraces.

    python tools/replay_verify.py trace.jsonl

Re-scores every early-exit evaluation of a GPU request trace with the
reference's own MetricQEvaluator + decide_exit (oracle/_ref/libmoaref.so,
compiled from /root/reference/proj/core; the mock embedding provider) over the
GPU's observed completion order -- the completing agents' literal output
tokens and logprobs carried in the trace -- and checks q (1e-9 relative),
the exit draw and the decision bit-exactly.  Also checks the trace's
structural invariants (agent records, pruned agents stopped early, the
e2e latency equals the last completion).  Test infrastructure: it links the
reference build, never the product."""
from __future__ import annotations

import ctypes
import json
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.rng import hash_combine  # noqa: E402


def _ref():
    lib = ctypes.CDLL(str(ROOT / "oracle" / "_ref" / "libmoaref.so"))
    lib.moaref_call.restype = ctypes.c_char_p
    lib.moaref_call.argtypes = [ctypes.c_char_p]
    return lambda req: json.loads(lib.moaref_call(json.dumps(req).encode()))


def parse(text: str):
    meta, agents, evals = None, {}, []
    for line in text.splitlines():
        if not line.strip():
            continue
        j = json.loads(line)
        if j["record"] == "meta":
            meta = j
        elif j["record"] == "agent":
            agents[j["agent"]] = j
        elif j["record"] == "metricq":
            evals.append(j)
    if meta is None:
        raise ValueError("trace: missing meta record")
    return meta, agents, evals


def verify(text: str, q_rtol: float = 1e-9) -> dict:
    meta, agents, evals = parse(text)
    call = _ref()
    master = hash_combine(meta["seed"], meta["sample_index"])
    by_group = defaultdict(list)
    for e in evals:
        if e["evaluated"]:
            by_group[e["group"]].append(e)
    checked, failures = 0, []
    for group, recs in by_group.items():
        recs.sort(key=lambda e: e["eval_index"])
        outs = [agents[e["completed"]]["output_token_ids"] for e in recs]
        lps = [agents[e["completed"]]["logprobs"] for e in recs]
        ref = call({"cmd": "metricq", "hidden": meta["provider"]["hidden"], "seed": meta["provider"]["seed"],
                    "tau": meta["tau"], "include_diagonal": meta["include_diagonal"], "rng_master": master,
                    "rng_label": group, "outputs": outs, "logprobs": lps})
        if "error" in ref:
            raise RuntimeError(f"reference metricq failed: {ref}")
        for e, r in zip(recs, ref["evals"]):
            checked += 1
            q, rq = e["score"]["q"], r["q"]
            if abs(q - rq) > q_rtol * max(1.0, abs(rq)) or e["decision"]["draw"] != r["draw"] or \
                    e["decision"]["exited"] != r["exited"]:
                failures.append({"group": group, "eval_index": e["eval_index"], "gpu": (q, e["decision"]),
                                 "reference": (rq, r["draw"], r["exited"])})
    # structural invariants
    last = max(a["complete_t"] for a in agents.values())
    if abs(last - meta["e2e_latency"]) > 1e-9:
        failures.append({"invariant": "e2e_latency == last complete_t", "last": last, "e2e": meta["e2e_latency"]})
    for name, a in agents.items():
        if a["pruned"] and a["invoked"] and a["decode_end"] >= 0:
            failures.append({"invariant": "pruned agents never reach decode_end", "agent": name})
    return {"evaluations_checked": checked, "groups": len(by_group), "failures": failures, "ok": not failures}


if __name__ == "__main__":
    res = verify(Path(sys.argv[1]).read_text())
    print(json.dumps(res, indent=1))
    sys.exit(0 if res["ok"] else 1)
