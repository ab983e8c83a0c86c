"""Debug: test_incremental_prefill_equals_one_shot under feature flags."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    from oracle import rng as orng
    from oracle.model import CpuModel, make_spec
    from oracle.parity import check_agent
    from paper_2512_18126_b200 import capi
    prompt = orng.synth_tokens(4, "p", 70)
    eng = capi.Engine([capi.model_spec("agg", "tiny", 2, max_agents=2)], max_ctx=1024, max_out=64)
    a, b = (1, 0), (1, 1)
    eng.add_agent(a, 0); eng.add_agent(b, 0)
    eng.generate(a, prompt, 16, 32)
    eng.prefill_only(b, 0, prompt[:30]); eng.step()
    eng.prefill_only(b, 30, prompt[30:61]); eng.step()
    eng.generate(b, prompt, 16, 32)
    while eng.busy():
        eng.step()
    ta, la, _ = eng.read_output(a, 16); tb, lb, _ = eng.read_output(b, 16)
    eng.close()
    model = CpuModel(make_spec("agg", "tiny", seed=2), 1024)
    res = []
    for toks, lps in ((ta, la), (tb, lb)):
        chk = check_agent(model, prompt, toks, lps)
        res.append({k: chk[k] for k in ("checked", "mismatches", "max_lp_err", "lp_ok")})
    print(json.dumps({"env": sys.argv[1], "a": res[0], "b": res[1], "ta": list(ta[:4]), "tb": list(tb[:4])}))
else:
    for env in ["", "MOA_DECODE_TMA=0", "MOA_EVICT_FIRST=0", "MOA_QKV_ATTN=0", "MOA_NORM_FOLD=0", "MOA_GRAPHS=0",
                "MOA_PREFILL_ATTN=0", "MOA_FUSE_O=0", "MOA_DECODE_RUN=1", "MOA_PREFILL_MIN_ROWS=100000"]:
        e = dict(os.environ)
        if env:
            k, v = env.split("=")
            e[k] = v
        subprocess.run([sys.executable, __file__, env or "default"], env=e)
