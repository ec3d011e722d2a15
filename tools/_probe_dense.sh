timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gt.log 2>&1; echo rc=$? >> gpurun_out/gt.log
for w in lasso_dense soc_ls logreg; do timeout 300 python tools/workload_probe.py $w 100 20000 2>&1 | tail -1; done > gpurun_out/dense_probe.log
timeout 300 python tools/dense_bench.py > gpurun_out/dense_bench.log 2>&1
