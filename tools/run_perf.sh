for e in 0 1 2; do echo "== CK_TC_EXP=$e"; CK_TC_EXP=$e python tools/gemm_exp.py; done
