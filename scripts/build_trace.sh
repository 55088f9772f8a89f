# debug build with %globaltimer phase stamps (PPFG_TRACE), selected via PPFG_SO
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -shared -DPPFG_TRACE -Iinclude -o paper_1411_3656_b200/libppfg_trace.so paper_1411_3656_b200/csrc/ppfg.cu
