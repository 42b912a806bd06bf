for fl in write read none; do python tools/edge_bench.py --configs C3,C4,MOB --flush $fl | sed "s/^/$fl /"; done > gpurun_out/ef.txt 2>&1
cat gpurun_out/ef.txt
