// C++ host-API drop-in check: the reference's frozen golden probe (test_swin_core.cpp:415-422)
// written against include/swinflow/b200.hpp exactly as the reference test is written against
// swin.hpp, running on the GPU in the FP32 validation mode. Prints y(1,77); exits non-zero on
// error (rc 4 without a GPU).
#include <cstdio>

#include "swinflow/b200.hpp"

using namespace swinflow;

int main(int argc, char** argv) {
    ModelConfig c;  // tiny_config(), test_swin_core.cpp:16-27
    c.hidden_dim = 16;
    c.n_heads = 4;
    c.ffn_dim = 32;
    c.n_layers = 2;
    c.window_px = 6;
    c.in_channels = 4;
    c.out_channels = 2;
    c.time_dim = 16;
    set_precision(argc > 1 ? std::atoi(argv[1]) : SWF_PREC_FP32);
    try {
        auto p = init_parameters_random<double>(c, 2024);
        MatX<double> x(c.in_channels, 144);
        for (i64 i = 0; i < x.size(); ++i) x.data()[i] = gaussian(2025, u64(i));
        const MatX<double> y = forward(p, x, 0.62831853071795862, 12, 12);
        std::printf("%.16f\n", y(1, 77));
        return 0;
    } catch (const DeviceError& e) {
        std::fprintf(stderr, "device error: %s\n", e.what());
        return 4;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
