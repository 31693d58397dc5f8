for lib in "" variants/libmk2_u1.so variants/libmk2_u2.so variants/libmk2_u8.so; do echo "== ${lib:-default(4)}"; MK2_LIB=$lib python tools/probe_small_batch.py 4096 2>&1 | sed -n '3p;5p;7p;8p'; done
