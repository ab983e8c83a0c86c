"""A/B timing of one config under several environment settings (each in a
fresh process): python tools/abrun.py C2 48 'MOA_MK=0' 'MOA_MK=1 MOA_MK_STAGES=4' ..."""
import os, subprocess, sys

name, out = sys.argv[1], int(sys.argv[2])
code = f"""
import sys
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS
cfg = dict(CONFIGS['{name}'])
if {out}: cfg['out_len'] = [{out}] * 3
eng, qc = capi.engine_for(cfg)
ts = []
for i in range(4):
    r = eng.run_query(qc, sample=i % 2, resolve=False, detail=False)
    ts.append(r['e2e_ms'])
print('RES', ' '.join('%.2f' % t for t in ts), 'ticks', r['ticks'], 'tokens', r['tokens'], 'host_ms %.1f' % r['host_ms'])
"""
for spec in sys.argv[3:]:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split('=')
        env[k] = v
    p = subprocess.run([sys.executable, '-c', code], env=env, capture_output=True, text=True, timeout=900)
    line = [l for l in p.stdout.splitlines() if l.startswith('RES')]
    print(f'{name} [{spec}]', line[0] if line else ('FAILED ' + p.stderr[-1500:]), flush=True)
