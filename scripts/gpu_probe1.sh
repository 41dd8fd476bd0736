mkdir -p gpurun_out/probe
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/build/probe_inflight scripts/probe_inflight.cu
timeout 600 scripts/build/probe_inflight > gpurun_out/probe/inflight.txt 2>&1; echo probe rc=$?
timeout 600 python scripts/latency_breakdown.py > gpurun_out/probe/breakdown.txt 2>&1; echo bd rc=$?
timeout 900 python -m pytest tests/test_cli.py -q -m gpu 2>&1 | tail -2
cat gpurun_out/probe/breakdown.txt
