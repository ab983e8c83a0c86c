"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/moa_b200.h declares, and its host-side routing (Topology, SlotPlan)
matches the reference's own outputs (tests/golden/, generated from the
reference) -- bit-exact, including the error classes."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2512_18126_b200 import capi

HEADER = Path(__file__).resolve().parents[1] / "include" / "moa_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(moa_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(capi.EXPORTED)
    assert capi.lib().moa_version().startswith(b"moa_b200")


def test_error_codes_and_messages():
    # null engine -> ValidationError (MOA_ERR_VALIDATION = reference exit code 2)
    rc = capi.lib().moa_engine_reset(None)
    assert rc == capi.MOA_ERR_VALIDATION
    assert b"null" in capi.lib().moa_last_error()


def topo_c(spec):
    widths = spec["widths"]
    kind = 1 if spec["kind"] == "all_to_all" else 0
    cs = None
    if kind == 0:
        if "cluster_sizes" in spec:
            sizes = [s for l in spec["cluster_sizes"] for s in l]
        else:
            br = spec.get("branching", [])
            sizes = [br[l] if l < len(br) else 0 for l in range(len(widths) - 1) for _ in range(widths[l + 1])]
        cs = (C.c_int * max(1, len(sizes)))(*sizes)
    w = (C.c_int * len(widths))(*widths)
    n_agents = sum(max(0, x) for x in widths)
    off = (C.c_int * (n_agents + 1))()
    pre = (C.c_int * 4096)()
    rc = capi.lib().moa_topology(kind, len(widths), w, cs, off, pre, 4096)
    return rc, list(off), list(pre)


def test_topology_matches_reference(golden):
    for c in golden("topology.json"):
        spec, out = c["spec"], c["out"]
        if spec["kind"] == "tree" and "branching" in spec and len(spec["branching"]) != len(spec["widths"]) - 1:
            continue  # the C-ABI takes flattened cluster sizes; branching-count errors are a tree() concern
        rc, off, pre = topo_c(spec)
        if "error" in out:
            assert rc == capi.MOA_ERR_VALIDATION, spec
            continue
        assert rc == 0, capi.lib().moa_last_error()
        names = [a for layer in out["layers"] for a in layer]
        for k, a in enumerate(names):
            got = [names[i] for i in pre[off[k]:off[k + 1]]]
            assert got == out["precursors"][a], (spec, a)


def make_plan(case):
    slots = case["slots"]
    sl = (C.c_int * max(1, len(slots)))(*[int(s["precursor"].split(":")[0]) for s in slots])
    sp = (C.c_int * max(1, len(slots)))(*[int(s["precursor"].split(":")[1]) for s in slots])
    seps = [t for s in slots for t in s["separator"]]
    st = (C.c_int32 * max(1, len(seps)))(*seps)
    sn = (C.c_int * max(1, len(slots)))(*[len(s["separator"]) for s in slots])
    pre = (C.c_int32 * max(1, len(case["prefix"])))(*case["prefix"])
    suf = (C.c_int32 * max(1, len(case["suffix"])))(*case["suffix"])
    h = C.c_void_p()
    me = [int(x) for x in case["self"].split(":")]
    capi.check(capi.lib().moa_slotplan_create(me[0], me[1], pre, len(case["prefix"]), sl, sp, st, sn, len(slots),
                                              suf, len(case["suffix"]), int(case["incremental"]), C.byref(h)))
    return h


def decode_actions(buf, n):
    out, i = [], 0
    kinds = {0: "prefill_only", 1: "generate", 2: "reclaim"}
    while i < n:
        k, s, m = buf[i], buf[i + 1], buf[i + 2]
        out.append({"kind": kinds[k], "start": s, "tokens": list(buf[i + 3:i + 3 + m])})
        i += 3 + m
    return out


def test_slotplan_matches_reference(golden):
    ops = {"start": 0, "chunk": 1, "done": 2, "cancelled": 3}
    for c in golden("slotplan.json"):
        case = c["case"]
        h = make_plan(case)
        try:
            steps = []
            for ev in case["events"]:
                p = [int(x) for x in ev.get("producer", "0:0").split(":")]
                toks = ev.get("tokens", [])
                tb = (C.c_int32 * max(1, len(toks)))(*toks)
                buf = (C.c_int32 * 8192)()
                n = C.c_int()
                rc = capi.lib().moa_slotplan_event(h, ops[ev["op"]], p[0], p[1], tb, len(toks), buf, 8192, C.byref(n))
                if rc != 0:
                    steps.append({"error": {capi.MOA_ERR_RUNTIME: "RunError",
                                            capi.MOA_ERR_VALIDATION: "ValidationError"}[rc]})
                    break
                steps.append({"actions": decode_actions(buf, n.value)})
            ref_steps = [{"error": s["error"]} if "error" in s else s for s in c["out"]["steps"]]
            assert steps == ref_steps, case
        finally:
            capi.lib().moa_slotplan_free(h)


@pytest.mark.parametrize("name", ["C0", "C1", "C1U", "C2", "C3", "C4-tree", "C4-dense", "C5"])
def test_query_config_marshalling(name):
    from paper_2512_18126_b200.configs import CONFIGS
    cfg = CONFIGS[name]
    q = capi.QueryConfig(cfg, {t: i for i, t in enumerate(cfg["models"])})
    assert q.c.n_layers == len(cfg["topology"]["widths"])
    assert q.c.mode == capi.MODES[cfg["mode"]]


def test_library_has_no_unresolved_internal_symbols():
    """Every moa:: symbol the library references is defined in it (dlopen with
    RTLD_NOW fails on the GPU box otherwise)."""
    import os
    import subprocess
    C.CDLL(str(capi.LIB_PATH), mode=os.RTLD_NOW)
    out = subprocess.run(["nm", "-D", "--undefined-only", str(capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "_ZN3moa" not in out, [l for l in out.splitlines() if "_ZN3moa" in l]
