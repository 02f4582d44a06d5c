set -x
timeout 300 python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
timeout 300 python bench.py --impl reference > gpurun_out/b_cfg2_ref.json 2> gpurun_out/b_cfg2_ref.err
timeout 300 python bench.py --workload cfg1 > gpurun_out/b_cfg1.json 2> gpurun_out/b_cfg1.err
timeout 300 python bench.py --workload cfg3 > gpurun_out/b_cfg3.json 2> gpurun_out/b_cfg3.err
timeout 400 python bench.py --workload cfg4 > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
timeout 600 python bench.py --workload cfg5 --steps 3 --e2e-steps 1 > gpurun_out/b_cfg5.json 2> gpurun_out/b_cfg5.err
timeout 600 python bench.py --workload cfg5 --steps 3 --e2e-steps 1 --slab --no-cpu-baseline > gpurun_out/b_cfg5_slab.json 2> gpurun_out/b_cfg5_slab.err
timeout 600 python bench.py --workload cfg5 --steps 3 --e2e-steps 1 --ring --no-cpu-baseline > gpurun_out/b_cfg5_ring.json 2> gpurun_out/b_cfg5_ring.err
timeout 300 python bench.py --mode fast --no-cpu-baseline > gpurun_out/b_cfg2_fast.json 2> gpurun_out/b_cfg2_fast.err
