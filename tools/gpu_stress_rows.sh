# stress runs after the tile-height change: the general mix at the default choice and with the
# float box kernel's tile height forced to 5 rows
O=gpurun_out/stressr; mkdir -p $O; rm -f $O/*
timeout 700 python tools/stress.py 540 5051 > $O/stress_5051.log 2>&1; echo "mix=$?" >> $O/status.txt
SC_BM_BOXF_ROWS=5 timeout 700 python tools/stress.py 540 5052 > $O/stress_rows5_5052.log 2>&1; echo "rows5=$?" >> $O/status.txt
