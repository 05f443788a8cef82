mkdir -p gpurun_out
D=paper_2506_06095_b200
( for v in emu1 emu2 sus200 sus2000; do echo "== ${v:-default}"; if [ -n "$v" ]; then export SF_B200_LIB=$D/_lib_$v/libsf_b200.so; else unset SF_B200_LIB; fi; timeout 300 python tools/attn_cfg.py cfg2 cfg3 cfg4 dense; done ) > gpurun_out/attn3_variants2.txt 2>&1
cat gpurun_out/attn3_variants2.txt
