for i in 1 2; do for G in 0 1; do QEFT_GROUPED=$G timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1 | sed "s/^/G=$G /"; done; done
