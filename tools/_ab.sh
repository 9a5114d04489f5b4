python tools/burst_ab.py exp/v/old.so exp/v/mb2.so exp/v/mb3.so exp/v/mb4.so
