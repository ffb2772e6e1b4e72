cd $GRAFT_REPO_ROOT
export ST_SANITIZER_OUT=gpurun_out/sanitizer
timeout 2400 python -m pytest tests/test_sanitizer.py -q -x --timeout 1800 > gpurun_out/g17_san.txt 2>&1
tail -20 gpurun_out/g17_san.txt
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|SYNCCHECK" gpurun_out/sanitizer/*.log | sort | uniq -c
