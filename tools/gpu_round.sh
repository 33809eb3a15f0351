#!/bin/bash
# one GPU session: tests, bench, launch list, ncu full captures of the sweep and the post kernels
# (outputs in gpurun_out/)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -n 5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-extras --no-cpu > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/ncu_sweep -f python tools/one_posterior.py c4 full > gpurun_out/ncu_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:post_gradB_blk_kernel -s 20 -c 1 -o gpurun_out/ncu_gradB -f python tools/one_posterior.py c4 full > gpurun_out/ncu_gradB.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cut_kernel -s 20 -c 1 -o gpurun_out/ncu_cut -f python tools/one_posterior.py c4 full > gpurun_out/ncu_cut.log 2>&1
ls -la gpurun_out/
