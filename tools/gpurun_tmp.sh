rm -f gpurun_out/sweep.txt
SCHEDS="880,960,8,4 800,950,8,4 750,930,8,4 700,900,8,4 650,900,8,4 600,880,8,4" bash tools/sweep_sched.sh --config c4
