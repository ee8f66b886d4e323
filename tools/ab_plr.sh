# A/B of PLR iteration timings between library builds on one box:
#   bash tools/ab_plr.sh "A B C" reps   (tools/lib<L>.so per label)
LABELS=${1:-"A B"}
REPS=${2:-1}
for r in $(seq 1 $REPS); do
for L in $LABELS; do
  AMZ_LIB_PATH=tools/lib$L.so python bench.py --no-cpu-baseline > gpurun_out/ab_$L.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab_$L.json'))
print('$L', ' '.join('%s=%.3f' % (k, d[k]['iteration_ms']) for k in ['parallel_plr','plr_perp','accel_perp','plr_parallel','accel_parallel']), 'accel_perp_replay=%.3f' % d['accel_perp']['replay_iteration_ms'])
"
done
done
