// C++ host-API checks on the GPU, written against include/swinflow/b200.hpp like the reference's
// tests are written against swin.hpp:
//  1. the reference-signature forward() on a single-process multi-device topology (window
//     parallelism 1x2, device_ids from argv: "0 0" on a 1-GPU box, "0 1" on two GPUs) equals the
//     single-device forward bitwise;
//  2. an in-place update of the caller's Parameters (what AdamW / EMA do, optim.hpp:59-106) is seen by
//     the next forward() (the context cache re-uploads changed parameters);
//  3. block_window_forward (swin.hpp:306-325) through the same API.
// Prints "GROUP_PROBE PASS" and exits 0 on success.
#include <cstdio>
#include <cstdlib>

#include "swinflow/b200.hpp"

using namespace swinflow;

int main(int argc, char** argv) {
    ModelConfig c;  // BASELINE configs[0]: 32x64 grid, 8 channels, 8x8 windows, 2 blocks, dim 128, 4 heads
    c.hidden_dim = 128;
    c.n_heads = 4;
    c.ffn_dim = 256;
    c.n_layers = 2;
    c.window_px = 8;
    c.in_channels = 8;
    c.out_channels = 3;
    c.time_dim = 128;
    const int H = 32, W = 64;
    const int d0 = argc > 2 ? std::atoi(argv[1]) : 0, d1 = argc > 2 ? std::atoi(argv[2]) : 0;
    try {
        auto p = init_parameters_random<float>(c, 2024, 0.05);
        MatX<float> x(c.in_channels, i64(H) * W);
        for (i64 i = 0; i < x.size(); ++i) x.data()[i] = float(gaussian(2025, u64(i)));
        set_precision(SWF_PREC_BF16);
        const MatX<float> y1 = forward(p, x, 0.7f, H, W);
        Topology t;
        t.wp_a = 1;
        t.wp_b = 2;
        t.device_ids = {d0, d1};
        set_topology(t);
        const MatX<float> y2 = forward(p, x, 0.7f, H, W);
        bool same = true;
        for (i64 i = 0; i < y1.size(); ++i) same &= y1.data()[i] == y2.data()[i];
        std::printf("group 1x2 on devices {%d,%d} bitwise == 1 device: %s\n", d0, d1, same ? "yes" : "NO");
        // in-place parameter update: the cached group context must re-upload
        for (i64 i = 0; i < p.blocks[0].w_out.size(); ++i) p.blocks[0].w_out.data()[i] *= 1.5f;
        const MatX<float> y3 = forward(p, x, 0.7f, H, W);
        set_topology(Topology{});
        release_contexts();
        const MatX<float> y4 = forward(p, x, 0.7f, H, W);  // fresh single-device context
        bool changed = false, fresh = true;
        for (i64 i = 0; i < y1.size(); ++i) {
            changed |= y3.data()[i] != y2.data()[i];
            fresh &= y3.data()[i] == y4.data()[i];
        }
        std::printf("in-place update seen: %s, equals a fresh context: %s\n", changed ? "yes" : "NO", fresh ? "yes" : "NO");
        // block_window_forward of block 1 (shifted) on window (3, 5): finite, changes the input
        MatX<float> xin(c.hidden_dim, i64(c.window_px) * c.window_px);
        for (i64 i = 0; i < xin.size(); ++i) xin.data()[i] = float(0.7 * gaussian(92, u64(i)));
        const MatX<float> xo = block_window_forward(p, 1, 0.6f, H, W, 3, 5, xin);
        double dmax = 0;
        bool finite = true;
        for (i64 i = 0; i < xo.size(); ++i) {
            finite &= std::isfinite(xo.data()[i]);
            dmax = std::max(dmax, double(std::fabs(xo.data()[i] - xin.data()[i])));
        }
        std::printf("block_window_forward: finite=%d max|dx|=%.4f\n", int(finite), dmax);
        const bool ok = same && changed && fresh && finite && dmax > 1e-3;
        std::printf("GROUP_PROBE %s\n", ok ? "PASS" : "FAIL");
        return ok ? 0 : 1;
    } catch (const DeviceError& e) {
        std::fprintf(stderr, "device error: %s\n", e.what());
        return 4;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
