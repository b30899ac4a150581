for cl in 2 8; do echo "cluster=$cl"; EIGMOD_OPTS=cluster=$cl python tools/exp_solver_share.py; done > gpurun_out/share.log 2>&1
