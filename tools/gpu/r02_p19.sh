timeout 900 python -m pytest tests/test_conformance.py tests/test_cli.py -q -p no:cacheprovider > gpurun_out/p19_tests.log 2>&1; echo tests rc=$?
tail -15 gpurun_out/p19_tests.log
./oracle/_ref/conformance/acceptance_test > gpurun_out/acceptance.txt 2>&1; echo acc rc=$?
grep -E "criterion|passed|FAILED|recovery|mean sweep" gpurun_out/acceptance.txt | head -40
./oracle/_ref/conformance/cli_test > gpurun_out/cli_test.txt 2>&1; echo cli rc=$?; tail -3 gpurun_out/cli_test.txt
