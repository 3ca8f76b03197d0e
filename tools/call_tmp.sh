python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for M in replica sections; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --mode $M --dist-backend gloo --no-e2e > gpurun_out/multi_$M.log 2>&1; echo "rc=$?" >> gpurun_out/multi_$M.log
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/ref.log 2>&1; echo "rc=$?" >> gpurun_out/ref.log
