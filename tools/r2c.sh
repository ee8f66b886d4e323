R=r2c
for m in "plr 2048" "accel 2048" "plr 16384"; do
  set -- $m
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launch_$1_$2.csv python tools/plr_profile.py $1 $2 > /dev/null 2>&1
done
echo done
