for v in old new old new; do python tools/variant_apply.py tools/var/lib_$v.so cfg4 6; done
