OOCNMF_PROFILE_IO=1 PYTHONPATH=. timeout 600 python tools/e2e_probe.py > gpurun_out/r3z_e2e_sparse.txt 2>&1
