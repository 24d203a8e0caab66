mkdir -p gpurun_out/rf2
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T --nproc-per-node 2 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 --config C3 > gpurun_out/rf2/n2c3.json 2> gpurun_out/rf2/n2c3.err
$T --nproc-per-node 2 --master-port 29532 bench.py --gpus 2 --steps 10 --warmup 3 --config C4 > gpurun_out/rf2/n2c4.json 2> gpurun_out/rf2/n2c4.err
$T --nproc-per-node 4 --master-port 29533 bench.py --gpus 4 --steps 10 --warmup 3 --config C4 > gpurun_out/rf2/n4c4.json 2> gpurun_out/rf2/n4c4.err
$T --nproc-per-node 4 --master-port 29534 bench.py --gpus 4 --steps 10 --warmup 3 --config C3 > gpurun_out/rf2/n4c3.json 2> gpurun_out/rf2/n4c3.err
$T --nproc-per-node 4 --master-port 29535 bench.py --gpus 4 --steps 10 --warmup 3 --config C5 > gpurun_out/rf2/n4c5.json 2> gpurun_out/rf2/n4c5.err
for f in n2c3 n2c4 n4c4 n4c3 n4c5; do echo "$f $(python -c "import json;d=json.loads(open('gpurun_out/rf2/$f.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), d['config']['batch'], d['config']['inflight'], d['clocks']['sm_mhz'])")"; done
