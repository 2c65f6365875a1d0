OOCNMF_PROFILE_IO=1 PYTHONPATH=. timeout 900 python tools/e2e_phase_probe.py > gpurun_out/r4f_e2e.txt 2>&1
