SWEEP_SRCS := sweep_f16_x1.cu sweep_f16_x2.cu sweep_f16_f64.cu sweep_bf16_x1.cu sweep_bf16_x2.cu sweep_bf16_f64.cu sweep_f32_x1.cu sweep_f32_x2.cu sweep_f32_f64.cu sweep_f64_f64.cu
