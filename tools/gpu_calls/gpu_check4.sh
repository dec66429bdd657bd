# parity + bench (x5k) + cfg4 bench (x20k) with the mesh-size team rule
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e-u8 > gpurun_out/b1.json 2> gpurun_out/b1.err
python -c "import json; d=json.load(open('gpurun_out/b1.json')); print('bench', round(d['value']), round(d['ms_per_step'],3), d['pcg_iter_us'])" || tail -3 gpurun_out/b1.err
timeout 400 python bench.py --preset x20k --gn 4 --pcg 8 --no-cpu-baseline > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err
python -c "import json; d=json.load(open('gpurun_out/cfg4.json')); print('cfg4', round(d['value']), round(d['ms_per_step'],3), d['pcg_iter_us'], d['e2e']['value'])" || tail -3 gpurun_out/cfg4.err
