for pf in 0 8 16 32 64; do echo "L2PF=$pf"; RAPDB_L2PF=$pf REPS=3 python tools/step_profile.py C1 2>&1 | grep "C1 mono"; done
for pf in 0 16 32; do echo "L2PF=$pf"; RAPDB_L2PF=$pf REPS=2 python tools/step_profile.py C4 nm 2>&1 | grep "C4 nm"; done
