# k_dyn / k_spec launch times per LPW (ncu launch list), HOME then RESAMPLE
for l in ${@:-4}; do
AMZ_DYN_LPW=$l ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lrm_$l.csv -k regex:"k_dyn|k_spec" python tools/rollout_modes.py > /dev/null 2>&1
done
