# GAE kernel-selection sweep at HBM-sized batches (see tools/gae_large.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/gae_exp3.log
: > $O
python tools/gae_large.py >> $O 2>&1
AMZ_GAE_KERNEL=7 python tools/gae_large.py 4096 8192 16384 65536 262144 >> $O 2>&1
AMZ_GAE_KERNEL=7 AMZ_GAE_M=2 python tools/gae_large.py >> $O 2>&1
AMZ_GAE_KERNEL=4 python tools/gae_large.py >> $O 2>&1
AMZ_GAE_KERNEL=7 timeout 600 python -m pytest tests -x -q -m gpu -k "gae or score or plr" >> $O 2>&1
AMZ_GAE_KERNEL=7 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gae --csv --log-file gpurun_out/gae_ncu_k7.csv python tools/gae_large.py 65536 > /dev/null 2>&1
AMZ_GAE_KERNEL=7 ncu --set full --import-source on --clock-control none -k regex:k_gae_score7 -s 2 -c 1 -o gpurun_out/gae7_full python tools/gae_large.py 65536 > /dev/null 2>&1
