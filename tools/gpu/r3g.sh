OOCNMF_PROFILE_IO=1 PYTHONPATH=. timeout 600 python tools/e2e_dense_probe.py > gpurun_out/r3g_e2e.txt 2>&1
