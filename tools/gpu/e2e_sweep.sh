for l in variants/lib_c1m.so paper_2306_05051_b200/libglint.so variants/lib_c128k.so; do
  GLINT_LIB=$PWD/$l timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$l', '%.4e' % e['value'], '%.3f' % e['h2d_frac'], e['h2d_gbs_measured_peak'])"
done
