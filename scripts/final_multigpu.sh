set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python bench.py > gpurun_out/fc5_n1.json 2> gpurun_out/fc5_n1.err
for n in 2 4; do $TR --nproc-per-node $n --master-port 2960$n bench.py --gpus $n > gpurun_out/fc5_n$n.json 2> gpurun_out/fc5_n$n.err; done
python bench.py --config CP --no-cpu-baseline > gpurun_out/fcp_n1.json 2>/dev/null
for n in 2 4; do $TR --nproc-per-node $n --master-port 2961$n bench.py --gpus $n --config CP --no-cpu-baseline > gpurun_out/fcp_n$n.json 2>/dev/null; done
for n in 2 4; do $TR --nproc-per-node $n --master-port 2962$n bench.py --gpus $n --config C4 --strong --no-cpu-baseline > gpurun_out/fc4s_n$n.json 2>/dev/null; done
python -m pytest tests/test_gpu_multigpu.py -q > gpurun_out/pytest_mg.log 2>&1
tail -2 gpurun_out/pytest_mg.log
