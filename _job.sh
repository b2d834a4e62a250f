mkdir -p gpurun_out/r2z
python bench.py > gpurun_out/r2z/bench.json 2> gpurun_out/r2z/bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2z/ref.json 2> gpurun_out/r2z/ref.err; echo ref=$?
NDG_PARITY_LOG=gpurun_out/r2z/parity_fullsize.jsonl python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r2z/fullsize.log 2>&1; echo full=$?
tail -1 gpurun_out/r2z/fullsize.log
