# final-code scaling on one 4-GPU box: C5 weak (1/2/4), C4 strong (1/2/4), CP weak (1/2/4)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python bench.py --no-cpu-baseline > gpurun_out/s_c5_n1.json 2>/dev/null
for n in 2 4; do $TR --nproc-per-node $n --master-port 2990$n bench.py --gpus $n --no-cpu-baseline > gpurun_out/s_c5_n$n.json 2>/dev/null; done
python bench.py --config C4 --strong --no-cpu-baseline > gpurun_out/s_c4s_n1.json 2>/dev/null
for n in 2 4; do $TR --nproc-per-node $n --master-port 2991$n bench.py --gpus $n --config C4 --strong --no-cpu-baseline > gpurun_out/s_c4s_n$n.json 2>/dev/null; done
python bench.py --config CP --no-cpu-baseline > gpurun_out/s_cp_n1.json 2>/dev/null
for n in 2 4; do $TR --nproc-per-node $n --master-port 2992$n bench.py --gpus $n --config CP --no-cpu-baseline > gpurun_out/s_cp_n$n.json 2>/dev/null; done
