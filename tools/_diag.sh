mkdir -p gpurun_out/tp8
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --inflight 2"
GH_SPLIT_NOWAIT=1 GH_PROFILE_GEMMS=2 timeout -k 20 400 $R --shard 149 > gpurun_out/tp8/t1_b447.json 2> gpurun_out/tp8/t1_b447.err
GH_SPLIT_NOWAIT=1 GH_PROFILE_GEMMS=2 timeout -k 20 400 $R --shard 192 --tier1-tp 2 > gpurun_out/tp8/tp2_b384.json 2> gpurun_out/tp8/tp2_b384.err
timeout -k 20 400 $R --tier1-tp 2 > gpurun_out/tp8/tp2_n4.json 2> gpurun_out/tp8/tp2_n4.err
timeout -k 20 400 $R --tier1-tp 2 --inflight 3 > gpurun_out/tp8/tp2_n4_if3.json 2> gpurun_out/tp8/tp2_n4_if3.err
for f in t1_b447 tp2_b384 tp2_n4 tp2_n4_if3; do echo "$f $(grep -h "rank 0 (t" gpurun_out/tp8/$f.err)"; tail -c 300 gpurun_out/tp8/$f.err | grep -i error; done
