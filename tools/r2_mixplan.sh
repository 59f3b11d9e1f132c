# planner cost-model sweep for the fused backward (C2, T = 8192): fused_us per setting
for dwk in 0.5 0.55 0.6 0.65 0.7; do for epd in 1.5 3; do
r=$(ROAST_MIX_DWK=$dwk ROAST_MIX_EPI_DX=$epd ROAST_VERBOSE=1 timeout 120 python tools/bwd_fused_probe.py 8192 2>&1)
echo "dwk $dwk epi_dx $epd $(echo "$r" | grep -o 'makespan [0-9.]*.*split [0-9]*') $(echo "$r" | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["fused_us"],1))')"
done; done
