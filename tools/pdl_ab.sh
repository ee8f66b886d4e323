cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/ab.log
for i in 1 2; do
  AMZ_NO_PDL=1 python bench.py --no-extra --steps 100 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nopdl', b['value'], b['e2e']['value'], b['e2e']['values_f32']['value'], b['e2e']['host_enqueue_ms_per_step'])" >> gpurun_out/ab.log
  python bench.py --no-extra --steps 100 2>/dev/null | python -c "import json,sys; b=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl  ', b['value'], b['e2e']['value'], b['e2e']['values_f32']['value'], b['e2e']['host_enqueue_ms_per_step'])" >> gpurun_out/ab.log
done
