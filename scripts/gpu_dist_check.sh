# torchrun + NCCL plumbing at world size 1 (forced all-gather + merge), the reference arm
# under torchrun, and ncu full captures of the cfg3 / cfg4 kernels.
mkdir -p gpurun_out/dist gpurun_out/ncu
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 20 --warmup 3 --force-collective --no-cpu > gpurun_out/dist/forced.json 2> gpurun_out/dist/forced.err
echo forced rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/dist/ref.json 2> gpurun_out/dist/ref.err
echo ref rc=$?
C3="python bench.py --config cfg3 --steps 5 --warmup 2 --no-e2e --no-cpu"
C4="python bench.py --config cfg4 --steps 5 --warmup 2 --no-e2e --no-cpu"
$C3 > gpurun_out/ncu/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaves -s 2 -c 1 -o gpurun_out/ncu/prof_cfg3 $C3 > gpurun_out/ncu/full3.log 2>&1; echo full3 rc=$?
$C4 > gpurun_out/ncu/plain4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaves -s 2 -c 1 -o gpurun_out/ncu/prof_cfg4 $C4 > gpurun_out/ncu/full4.log 2>&1; echo full4 rc=$?
python - <<'PY'
import json
for f in ("gpurun_out/dist/forced.json", "gpurun_out/dist/ref.json"):
    try:
        d = json.load(open(f)); print(f, d["value"], d.get("gpu_launches"), d.get("config", {}).get("parallelism"), d.get("impl"))
    except Exception as e:
        print(f, "ERR", e)
PY
tail -3 gpurun_out/dist/forced.err
