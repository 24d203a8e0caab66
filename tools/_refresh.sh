mkdir -p gpurun_out/rf
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
$T --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/rf/n2.json 2> gpurun_out/rf/n2.err
$T --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/rf/n4.json 2> gpurun_out/rf/n4.err
$T --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --steps 10 --warmup 3 --shard 128 --inflight 5 > gpurun_out/rf/n4opt.json 2> gpurun_out/rf/n4opt.err
$T --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --steps 10 --warmup 3 --config C5 --tier1-tp 2 > gpurun_out/rf/c5_tp2.json 2> gpurun_out/rf/c5_tp2.err
$T --nproc-per-node 4 --master-port 29525 bench.py --gpus 4 --steps 10 --warmup 3 --config C3 --paged > gpurun_out/rf/n4c3p.json 2> gpurun_out/rf/n4c3p.err
for f in n2 n4 n4opt c5_tp2 n4c3p; do echo "$f $(python -c "import json;d=json.loads(open('gpurun_out/rf/$f.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), round(d['e2e']['value']), d['clocks']['sm_mhz'])")"; done
