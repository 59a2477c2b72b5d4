O=gpurun_out/c43; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/old.csv python _ab_old/ft_step_old.py --blocks 4 --steps 1 > /dev/null 2>&1; echo old $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/new.csv python scripts/ft_step.py --blocks 4 --steps 1 > /dev/null 2>&1; echo new $?
ls -la $O
