ROUNDS=5 python tools/burst_ab.py exp/v/base.so exp/v/y3.so exp/v/ch2.so exp/v/m331.so exp/v/fm0.so exp/v/y3ch2.so exp/v/t128.so exp/v/t512.so
