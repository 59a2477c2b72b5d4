O=gpurun_out/c40; mkdir -p $O
for i in 1 2; do
(cd _ab_old && timeout 600 python bench.py --no-cpu --no-dstep --no-sweep > ../$O/old.json 2>../$O/old.err); python -c "
import json; d=json.load(open('$O/old.json')); ft=d['finetune']; print('OLD r02', round(ft['value']), round(ft['ms_per_step'],2), round(d['value']))"
timeout 600 python bench.py --no-cpu --no-dstep --no-sweep > $O/new.json 2>$O/new.err; python -c "
import json; d=json.load(open('$O/new.json')); ft=d['finetune']; print('NEW', round(ft['value']), round(ft['ms_per_step'],2), round(d['value']))"
done
timeout 200 python scripts/ab_gemm.py 2>&1 | tail -1
