cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/ab
python bench.py --n 2048 --config 5 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab/base_2048.json 2>&1
for d in variants/*/; do v=$(basename $d); ARENA_FFT_LIB_DIR=$PWD/variants/$v/lib python bench.py --n 2048 --config 5 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab/${v}_2048.json 2>&1; done
python tools/ab_summary.py gpurun_out/ab/*_2048.json
