for i in 1 2; do
timeout 600 python _ab_old/ft_step_old.py --steps 5 2>&1 | tail -1 | sed 's/^/OLD /'
timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1 | sed 's/^/NEW /'
done
