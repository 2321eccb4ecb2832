for i in 1 2; do python tools/profile_sweep.py C1 30; done
