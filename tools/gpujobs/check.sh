timeout 1500 python -m pytest tests -m gpu -q -p timeout --timeout=600 -rf > gpurun_out/ck_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ck_pytest.log
timeout 600 tests/dropin/dropin_unit_tests > gpurun_out/ck_dropin.log 2>&1; echo "dropin rc=$?" >> gpurun_out/ck_dropin.log
