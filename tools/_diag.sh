for f in 0 1; do echo "flags=$f: $(GH_ATTN_FLAGS=$f timeout -k 10 120 python tools/attn_bench.py 64 512 2>&1 | tail -1)"; done
for f in 0 1; do echo "flags=$f 2048: $(GH_ATTN_FLAGS=$f timeout -k 10 120 python tools/attn_bench.py 64 2048 2>&1 | tail -1)"; done
echo "70b 256x512: $(timeout -k 10 120 python tools/attn_bench.py 256 512 70b 2>&1 | tail -1)"
