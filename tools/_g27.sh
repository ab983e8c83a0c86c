timeout 900 python -m paper_2512_18126_b200.ablation --base C5 --samples 3 --no-second-layer --json gpurun_out/ablation_c5.json 2>&1 | tail -8
