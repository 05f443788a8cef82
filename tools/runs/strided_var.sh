D=paper_2506_06095_b200
for v in "" snc snl; do echo "== ${v:-default}"; if [ -n "$v" ]; then export SF_B200_LIB=$D/_lib_$v/libsf_b200.so; else unset SF_B200_LIB; fi
timeout 300 python tools/strided_time.py 2>&1 | grep -E "bs8 n2048|n8192"
done
