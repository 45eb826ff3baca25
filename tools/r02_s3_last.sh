#!/bin/bash
mkdir -p gpurun_out
T=${1:-r02s3ar}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); print('bench', round(d['ms_per_step'],3), round(d['value']), d['config']['residual'], d['e2e']['seconds_per_step'], d['cpu_baseline']['value'], d['clocks'])"
timeout 900 python bench.py --config c3 --steps 10 --e2e-steps 3 > gpurun_out/${T}_c3.json 2> gpurun_out/${T}_c3.err
timeout 600 python bench.py --config c2 --steps 20 --e2e-steps 3 > gpurun_out/${T}_c2.json 2> gpurun_out/${T}_c2.err
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
tail -2 gpurun_out/${T}_pytest.log
timeout 900 python -m pytest oracle/_ref/h2ulv_suite/tests -q -p no:cacheprovider > gpurun_out/${T}_refsuite.log 2>&1
tail -1 gpurun_out/${T}_refsuite.log
