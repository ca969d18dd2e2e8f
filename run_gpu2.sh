for i in 1 2; do
for lib in ablib/lib_st2.so paper_2511_15076_b200/_lib/libginsim_b200.so; do
GINSIM_LIB=$PWD/$lib timeout 300 python bench.py --no-extras --no-e2e --no-cpu-baseline --steps 30 > gpurun_out/ab.log 2>&1
grep -h '^{' gpurun_out/ab.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('n1 $lib', {k:round(d.get(k),1) for k in ['us_per_step','dispatch_us','combine_us']})
"
GINSIM_LIB=$PWD/$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --no-extras --no-e2e --steps 30 > gpurun_out/ab2.log 2>&1
grep -h '^{' gpurun_out/ab2.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('n2 $lib', {k:round(d.get(k),1) for k in ['us_per_step','dispatch_us','combine_us']})
"
done; done
