cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q -k "headline" -s > gpurun_out/t_headline.log 2>&1; echo "headline rc=$?" >> gpurun_out/t_headline.log
python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; echo "gpu rc=$?" >> gpurun_out/t_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?" >> gpurun_out/bench1.err
