set -x
python bench.py --nx 256 --steps 6 --warmup 3 --no-cpu > gpurun_out/dd_n1.log 2>&1
CSN_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --nx 256 --steps 6 --warmup 3 > gpurun_out/dd_n2.log 2>&1
CSN_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --nx 256 --steps 6 --warmup 3 > gpurun_out/dd_n4.log 2>&1
CSN_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 8 --nx 256 --steps 6 --warmup 3 > gpurun_out/dd_n8.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/dd_tr1.log 2>&1
tail -c 600 gpurun_out/dd_n1.log gpurun_out/dd_n2.log gpurun_out/dd_n8.log
