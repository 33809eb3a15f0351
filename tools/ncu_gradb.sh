mkdir -p gpurun_out
export SCRF_OVERLAP=-1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:post_gradB_blk_kernel -c 1 -o gpurun_out/r02_gradB_v2 -f python tools/one_posterior.py c4 full > gpurun_out/ncu_gradB.log 2>&1
ls -la gpurun_out/r02_gradB_v2.ncu-rep
