timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | head -1
python - <<'PY'
import cProfile, pstats, os, sys, io
sys.argv=['c5_phases.py']
pr=cProfile.Profile()
src=open('tools/c5_phases.py').read()
src=src.replace('P.update_batch(st, g, batch); t.append','pr.enable(); P.update_batch(st, g, batch); pr.disable(); t.append')
exec(compile(src,'c5','exec'), {'__name__':'__main__','pr':pr,'__file__':os.path.abspath('tools/c5_phases.py')})
s=io.StringIO(); pstats.Stats(pr,stream=s).sort_stats('cumulative').print_stats(14); print(s.getvalue()[-2500:])
PY
