# A/B of the rollout between library builds on one box (tools/lib<L>.so per label):
#   bash tools/ab_render.sh "A B" reps
LABELS=${1:-"A B"}
REPS=${2:-2}
for r in $(seq 1 $REPS); do
for L in $LABELS; do
  AMZ_LIB_PATH=tools/lib$L.so python tools/rollout_large.py 65536 8 | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$L large rollout_ms %.4f frac %.4f' % (d['rollout_ms'], d['frac']))"
  AMZ_LIB_PATH=tools/lib$L.so python bench.py --no-cpu-baseline --no-extra --steps 30 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$L config2 ms %.4f roll %.4f' % (d['ms_per_step'], d['roofline']['kernel_ms']))"
done
done
