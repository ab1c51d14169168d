mkdir -p gpurun_out
for b in 8 16 24 32 48; do echo B=$b; MORAP_QP_B=$b python scripts/qp_probe.py --profile c4 231; done
