for cfg in C2 C3 C4; do python tools/time_stage.py $cfg staged 4 50; done
