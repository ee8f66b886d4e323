# per-launch k_plr_update times (us) of tools/plr_profile.py MODE N for each library label
MODE=$1; N=$2; shift 2
for L in "$@"; do
  echo $L $(AMZ_LIB_PATH=tools/lib$L.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_plr_update --csv python tools/plr_profile.py $MODE $N 2>/dev/null | grep k_plr_update | awk -F, '{v=$NF; gsub(/"/,"",v); printf "%d ", v/1000}')
done
