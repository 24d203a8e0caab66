cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > $O/n1.json 2> $O/n1.err; echo "n1 rc=$?"; cat $O/n1.json
timeout 400 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"; cat $O/ref.json
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > $O/n2.json 2> $O/n2.err; echo "n2 rc=$?"; cat $O/n2.json
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > $O/n4.json 2> $O/n4.err; echo "n4 rc=$?"; cat $O/n4.json
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --config C3 > $O/n4c3.json 2> $O/n4c3.err; echo "n4c3 rc=$?"; cat $O/n4c3.json
timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 4 --config C3 --paged > $O/n4c3_paged.json 2> $O/n4c3_paged.err; echo "n4c3p rc=$?"; cat $O/n4c3_paged.json
