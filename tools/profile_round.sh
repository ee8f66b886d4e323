# Round profile capture: bench line, reference arm line, launch list, ncu --set full of our kernels.
set -x
R=${1:-r1k}
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dyn|k_render|k_gae_score|k_spec|k_sample_levels_w|k_env_reset" \
    --launch-skip 8 -c 4 -o gpurun_out/${R}_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_plr_update|k_plr_sample" -c 4 \
    -o gpurun_out/${R}_plr_full python tools/plr_update_micro.py > /dev/null 2>&1

# large-batch GAE kernel (65536 lanes) launch times + one full capture
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gae \
    --csv --log-file gpurun_out/${R}_gae_large.csv python tools/gae_large.py 65536 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gae_score7 -s 2 -c 1 \
    -o gpurun_out/${R}_gae_large_full python tools/gae_large.py 65536 > /dev/null 2>&1
echo done
