timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2 c5; do timeout 600 python -c "
import sys; sys.path.insert(0,'.')
from paper_1811_07717_b200 import synthetic
from paper_1811_07717_b200.engine import EegEngine
from paper_1811_07717_b200.device import PcgOperator
p=synthetic.eeg_problem('$c', device=True)
e=EegEngine(p.mesh,p.electrodes,p.G,B=p.B,C=p.C,R=p.R)
op=PcgOperator(e.assemble())
print('$c', 'bandwidth', op.bandwidth, 'batch', op.batch_width(p.B.shape[1], 64))
" 2>&1 | tail -1; done
timeout 1500 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['pcg_iterations'],d['roofline']['kernels'],d['roofline']['pcg_round'])"
