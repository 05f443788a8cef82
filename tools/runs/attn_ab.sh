# A/B of attention library variants (attn_cfg shapes): usage bash tools/runs/attn_ab.sh base v1 v2 ... ("" = default)
D=paper_2506_06095_b200
for v in "$@"; do echo "== ${v:-default}"; if [ -n "$v" ] && [ "$v" != default ]; then export SF_B200_LIB=$D/_lib_$v/libsf_b200.so; else unset SF_B200_LIB; fi
timeout 300 python tools/attn_cfg.py cfg2 cfg3 cfg4 dense
done
