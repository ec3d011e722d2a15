for g in 148 96 64 32 16 8; do echo "G=$g"; CGB_GRID=$g timeout 120 python tools/workload_probe.py lasso_dense 300 5000 --profile 2>&1 | tail -2; done > gpurun_out/gs_lasso.log
for g in 148 64 32; do echo "G=$g"; CGB_GRID=$g timeout 120 python tools/workload_probe.py soc_ls 100 2000 2>&1 | tail -1; done > gpurun_out/gs_socls.log
