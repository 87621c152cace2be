# multi-GPU equivalence on 4 GPUs with z-decomposed grids (the 8-GPU grid (2, 2, 2) decomposes z too)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
p=29741
for g in 1,2,2 1,1,4; do
  echo "CP grid $g"
  ALG_GRID=$g $TR --master-port $p scripts/check_multigpu.py CP 2>/dev/null | grep '^{' | tail -1
  p=$((p + 1))
done
echo "C2 grid 1,2,2"
ALG_GRID=1,2,2 $TR --master-port $p scripts/check_multigpu.py C2 2>/dev/null | grep '^{' | tail -1
