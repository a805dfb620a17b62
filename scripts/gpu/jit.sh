for v in r1 ""; do echo "variant [$v]"; FM_LIB_VARIANT=$v python scripts/plan_jitter.py 4 | tail -2; done
echo "max threshold"; FM_POOL_RELEASE_BYTES=18446744073709551615 python scripts/plan_jitter.py 4 | tail -2
