timeout 600 python tools/tune_nd.py c5 f64 "[2]" '[{}, {"SB200_3D_GEO": 2}, {"SB200_3D_ITEMS_PER_CTA": 8}, {"SB200_3D_ITEMS_PER_CTA": 16}]' 100 > gpurun_out/tune_t.log 2>&1
timeout 600 python tools/tune_nd.py c5 f32 "[2]" '[{}, {"SB200_3D_GEO": 1}, {"SB200_3D_ITEMS_PER_CTA": 8}, {"SB200_3D_ITEMS_PER_CTA": 16}]' 100 >> gpurun_out/tune_t.log 2>&1
