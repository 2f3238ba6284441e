# ncu --set full of both two-pass sweep kernels at HEAD (n = 1e5 stored C) -> profiles/r02_head_ncu/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02_head_ncu
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:rowpass_tma_kernel|colpass_kernel" -c 2 \
   -o /tmp/sweep_head python tools/profile_sweep.py --n 100000 --iters 1 > gpurun_out/r02_head_ncu/ncu.log 2>&1
bash tools/ncu_extract.sh /tmp/sweep_head.ncu-rep gpurun_out/r02_head_ncu/sweep_head
