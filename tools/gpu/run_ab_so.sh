cp paper_2404_09544_b200/libgnnv.so /tmp/libgnnv_cur.so
cp paper_2404_09544_b200/gnnv.py /tmp/gnnv_cur.py
for rep in 1 2; do
for v in cur prev; do
cp /tmp/libgnnv_cur.so paper_2404_09544_b200/libgnnv.so
cp /tmp/gnnv_cur.py paper_2404_09544_b200/gnnv.py
[ $v = prev ] && cp tools/gpu/libgnnv_prev.so paper_2404_09544_b200/libgnnv.so && cp tools/gpu/gnnv_prev.py paper_2404_09544_b200/gnnv.py
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abso_$v.json 2>gpurun_out/abso.err || tail -3 gpurun_out/abso.err
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-pipeline > gpurun_out/abso_s_$v.json 2>>gpurun_out/abso.err
python -c "import json; d=json.load(open('gpurun_out/abso_$v.json')); e=json.load(open('gpurun_out/abso_s_$v.json')); print('$v rep$rep', round(d['ms_per_step'],4), round(e['ms_per_step'],4), {k: round(v*1000,1) for k,v in e['phases_ms_per_step'].items() if k in ('spmm_fwd.l1','spmm_fwd.l2')})"
done
done
cp /tmp/libgnnv_cur.so paper_2404_09544_b200/libgnnv.so
cp /tmp/gnnv_cur.py paper_2404_09544_b200/gnnv.py
