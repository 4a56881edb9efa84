mkdir -p gpurun_out
rm -f gpurun_out/nb_sweep.jsonl
for nb in 16 32 24 16; do
  python bench.py --steps 4 --warmup 2 --no-e2e --no-cpu --no-extras --nb $nb 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'nb': $nb, 'ms': d['ms_per_step'], 'pass': d['stages_ms']['pass_total'], 'qrcp': d['stages_ms']['qrcp'], 'err': d['rel_err_fro'], 'mhz': d['clocks']['sm_mhz'], 'design': d['roofline']['design_over_algorithmic']}))" >> gpurun_out/nb_sweep.jsonl
done
