# BASELINE configs[0..2] on one B200 through bench.py (performance lines beside the 512^3 headline)
mkdir -p gpurun_out
timeout 300 python bench.py --reso 32 --obj bulk --vol 0.2 --steps 5 --warmup 3 --no-ref-precision > gpurun_out/r02t_c0.json 2> gpurun_out/r02t_c0.err; echo c0 rc $?
timeout 600 python bench.py --reso 128 --obj shear --vol 0.2 --steps 20 --warmup 5 --no-ref-precision > gpurun_out/r02t_c1.json 2> gpurun_out/r02t_c1.err; echo c1 rc $?
timeout 900 python bench.py --reso 256 --obj bulk --vol 0.3 --steps 20 --warmup 5 --no-ref-precision > gpurun_out/r02t_c2.json 2> gpurun_out/r02t_c2.err; echo c2 rc $?
