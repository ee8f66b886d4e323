# Round profile capture: GPU tests, bench line, reference arm line, launch lists, ncu --set full
# of the headline kernels (config 2 and the 65536-lane roofline point) and of the PLR update.
R=${1:-r2x}
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${R}_pytest.log 2>&1; tail -3 gpurun_out/${R}_pytest.log
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
python tools/bw_probe.py > gpurun_out/${R}_bw.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dyn|k_render|k_gae_score|k_env_reset" \
    --launch-skip 4 -c 4 -o gpurun_out/${R}_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_dyn|k_render|k_env_reset" \
    --csv --log-file gpurun_out/${R}_large_launches.csv python tools/rollout_large.py 65536 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dyn|k_render" -s 2 -c 2 \
    -o gpurun_out/${R}_large_full python tools/rollout_large.py 65536 3 > /dev/null 2>&1
for m in "plr 2048" "accel 2048" "plr 16384"; do
  set -- $m
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_plr_$1_$2.csv python tools/plr_profile.py $1 $2 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_plr_update" -s 5 -c 1 \
    -o gpurun_out/${R}_plr_update_full python tools/plr_profile.py plr 2048 > /dev/null 2>&1
echo done
