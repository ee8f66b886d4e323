# GAE kernel-selection sweep at HBM-sized batches (see tools/gae_large.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
O=gpurun_out/gae_exp4.log
: > $O
python tools/gae_large.py 4096 16384 65536 262144 >> $O 2>&1
GAE_V32=1 python tools/gae_large.py 4096 16384 65536 262144 >> $O 2>&1
