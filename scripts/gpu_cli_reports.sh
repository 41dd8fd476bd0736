# The reference's experiment CLI on the GPU path (drop-in demonstration), reports into gpurun_out/cli/.
mkdir -p gpurun_out/cli
M="python -m paper_1401_0248_b200"
$M selftest --no-meta > gpurun_out/cli/selftest.md 2>&1; echo selftest rc=$?
$M hours100 --no-meta > gpurun_out/cli/hours100_seq.md 2>&1; echo hours100 rc=$?
$M hours100 --flavor cuda --no-meta > gpurun_out/cli/hours100_cuda.md 2>&1; echo hours100 cuda rc=$?
$M accuracy --no-meta > gpurun_out/cli/accuracy.md 2>&1; echo accuracy rc=$?
$M scaling --no-meta > gpurun_out/cli/scaling.md 2>&1; echo scaling rc=$?
$M bench --dot --repetitions 10 --no-meta > gpurun_out/cli/bench_dot.md 2>&1; echo bench rc=$?
$M read-baseline --channels 2 --no-meta > gpurun_out/cli/read2.md 2>&1; echo read rc=$?
$M noread-baseline --no-meta > gpurun_out/cli/noread.md 2>&1; echo noread rc=$?
