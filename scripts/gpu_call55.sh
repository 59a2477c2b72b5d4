O=gpurun_out/c55; mkdir -p $O
for n in 1 8 16; do
timeout 600 ncu --set full --clock-control none -k regex:gemv2_kernel -s 2 -c 1 -o $O/gu_n$n python scripts/prof_decode.py gate_up $n > /dev/null 2>&1
ncu -i $O/gu_n$n.ncu-rep --page raw --csv > $O/gu_n${n}_raw.csv
done
ls $O
