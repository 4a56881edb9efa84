# A/B of two builds on the same box: libmpid_ab.so (A, committed) vs libmpid.so (B, working tree)
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
for rep in 1 2; do
  for lib in libmpid_ab.so libmpid.so; do
    MPID_LIB=$lib python bench.py --steps 4 --warmup 2 --no-e2e --no-cpu --no-extras 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$lib', 'ms': d['ms_per_step'], 'pass': d['stages_ms']['pass_total'], 'qrcp': d['stages_ms']['qrcp'], 'mhz': d['clocks']['sm_mhz']}))" >> gpurun_out/ab.jsonl
  done
done
