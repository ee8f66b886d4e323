cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
AMZ_GAE_KERNEL=5 AMZ_GAE_M=4 AMZ_GAE_U=16 ncu --set full --import-source on --clock-control none -k regex:k_gae_score5 -s 2 -c 1 -o gpurun_out/gae5_full python tools/gae_large.py 65536 > gpurun_out/ncu5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gae_score2 -s 2 -c 1 -o gpurun_out/gae2_full python tools/gae_large.py 65536 >> gpurun_out/ncu5.log 2>&1
