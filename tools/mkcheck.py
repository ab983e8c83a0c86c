"""A/B: persistent decode megakernel (MOA_MK=1) vs per-op kernels (MOA_MK=0)
on C1 (tiny) and a short C2 (1b): timing, token agreement, oracle check."""
import json, os, subprocess, sys
sys.path.insert(0, '/root/repo')

def run(mk, name, out, var='MOA_MK'):
    code = f"""
import json, sys
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS
cfg = dict(CONFIGS['{name}'])
if {out}: cfg['out_len'] = [{out}] * 3
eng, qc = capi.engine_for(cfg)
res = []
for i in range(3):
    r = eng.run_query(qc, sample=i % 2, resolve=True, detail=True)
    res.append(dict(e2e_ms=r['e2e_ms'], ticks=r['ticks'], tokens=r['tokens'],
                    agents={{k: dict(output=v['output'], logprobs=[float(x) for x in v['logprobs']], prompt=v['prompt']) for k, v in r['agents'].items()}}))
print('JSON' + json.dumps(res))
"""
    env = dict(os.environ, **{var: str(mk)})
    p = subprocess.run([sys.executable, '-c', code], env=env, capture_output=True, text=True, timeout=600)
    if p.returncode != 0:
        print(name, 'mk', mk, 'FAILED', p.returncode, p.stderr[-3000:], p.stdout[-2000:])
        return None
    line = [l for l in p.stdout.splitlines() if l.startswith('JSON')][0]
    return json.loads(line[4:])

VAR = sys.argv[1] if len(sys.argv) > 1 else 'MOA_MK'
for name, out in (('C1', 0), ('C2', 48)):
    a = run(0, name, out, VAR)
    b = run(1, name, out, VAR)
    if not a or not b:
        continue
    print(name, VAR, '=0 e2e_ms', [round(x['e2e_ms'], 2) for x in a], '=1 e2e_ms', [round(x['e2e_ms'], 2) for x in b])
    ra, rb = a[-1], b[-1]
    same = sum(ra['agents'][k]['output'] == rb['agents'][k]['output'] for k in ra['agents'])
    first_diff = {k: next((i for i, (x, y) in enumerate(zip(ra['agents'][k]['output'], rb['agents'][k]['output'])) if x != y), None) for k in ra['agents']}
    print(name, f'agents with identical tokens {same}/{len(ra["agents"])}', 'first diff', first_diff)
    if name == 'C1':
        from oracle.model import CpuModel, make_spec
        from oracle.parity import check_agent
        from paper_2512_18126_b200.configs import C1
        for k, ag in rb['agents'].items():
            tag = C1['assign'][min(int(k[0]) - 1, 2)][0]
            mm = C1['models'][tag]
            chk = check_agent(CpuModel(make_spec(tag, mm['shape'], seed=mm['seed']), 1024), ag['prompt'], ag['output'], ag['logprobs'])
            print('  oracle', k, 'checked', chk['checked'], 'mismatches', chk['mismatches'], 'max_lp_err', round(chk['max_lp_err'], 4))
