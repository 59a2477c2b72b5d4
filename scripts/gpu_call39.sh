O=gpurun_out/c39; mkdir -p $O
(cd _ab_old && timeout 600 python bench.py --no-cpu --no-dstep --no-sweep > ../$O/old.json 2>../$O/old.err); python -c "
import json; d=json.load(open('$O/old.json')); ft=d['finetune']; print('OLD r02', round(ft['value']), round(ft['ms_per_step'],2), round(d['value']))"
timeout 600 python bench.py --no-cpu --no-dstep --no-sweep > $O/new.json 2>$O/new.err; python -c "
import json; d=json.load(open('$O/new.json')); ft=d['finetune']; print('NEW', round(ft['value']), round(ft['ms_per_step'],2), round(d['value']))"
