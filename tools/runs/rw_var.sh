D=paper_2506_06095_b200
for v in "" rw4 rw6; do echo "== ${v:-default}"; if [ -n "$v" ]; then export SF_B200_LIB=$D/_lib_$v/libsf_b200.so; else unset SF_B200_LIB; fi
timeout 300 python tools/rw_time.py 2>&1 | grep -E "band +(1|4|16):|p 0.00[25]|p 0.010"
done
