timeout 1500 python tools/paper_experiments.py --serial --out gpurun_out/paper_serial_accuracy.json 2>&1 | tail -3
