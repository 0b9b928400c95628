// Export-format fixtures from the reference itself:
// dataset.cpp's write_disparity_png quantisation (its PNG encoder is replaced
// by oracle/io_shim.cpp, which records the 16-bit image handed to it: libpng
// is not in this image) and write_boxes' text. Built and run by
// tests/golden/make_golden_export.py; writes a record stream to argv[1]:
//   name\0 dtype\0 i32 ndim, i64 dims[ndim], u64 bytes, raw bytes
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsgm/dataset.hpp"

namespace tsgm_shim {
extern tsgm::Image<std::uint16_t> last16;
}

static FILE* g_out;

static void rec(const std::string& name, const char* dtype, std::vector<uint32_t> dims,
                const void* data, size_t bytes) {  // make_golden.py's record format
    std::fwrite(name.c_str(), 1, name.size() + 1, g_out);
    std::fwrite(dtype, 1, std::strlen(dtype) + 1, g_out);
    const int32_t nd = static_cast<int32_t>(dims.size());
    std::fwrite(&nd, 4, 1, g_out);
    for (uint32_t d : dims) {
        const int64_t d64 = d;
        std::fwrite(&d64, 8, 1, g_out);
    }
    const uint64_t nb = bytes;
    std::fwrite(&nb, 8, 1, g_out);
    std::fwrite(data, 1, bytes, g_out);
}

static void rec_text(const std::string& name, const std::string& t) {
    rec(name, "u1", {static_cast<uint32_t>(t.size())}, t.data(), t.size());
}

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    g_out = std::fopen(argv[1], "wb");
    const std::string tmp = argv[2];
    std::mt19937 rng(1809);
    // f64 disparity maps: zeros (invalid), fractional values incl. exact .5/256 ties
    for (int c = 0; c < 3; ++c) {
        const int w = 37 + 11 * c, h = 23 + 5 * c;
        tsgm::Image<double> disp(w, h, 0.0);
        std::uniform_real_distribution<double> u(0.002, 255.99);
        std::uniform_int_distribution<int> k(0, 4);
        for (int i = 0; i < w * h; ++i) {
            const int kind = k(rng);
            double v = kind == 0 ? 0.0 : u(rng);
            if (kind == 1) v = (std::floor(v * 256.0) + 0.5) / 256.0;  // rounding tie
            if (kind == 2) v = std::floor(v);                          // integer disparity
            disp.data()[i] = v;
        }
        tsgm::write_disparity_png(tmp + "/d.png", disp);
        const std::string p = "f64_" + std::to_string(c);
        rec(p + "__disp", "f8", {static_cast<uint32_t>(h), static_cast<uint32_t>(w)}, disp.data(),
            8 * static_cast<size_t>(w) * h);
        rec(p + "__raw", "u2", {static_cast<uint32_t>(h), static_cast<uint32_t>(w)},
            tsgm_shim::last16.data(), 2 * static_cast<size_t>(w) * h);
    }
    // DisparityMap (integer WTA / export maps)
    for (int c = 0; c < 2; ++c) {
        const int w = 64 + 13 * c, h = 31 + 7 * c;
        tsgm::DisparityMap dm;
        dm.d = tsgm::Image<int32_t>(w, h, 0);
        dm.valid = tsgm::Image<uint8_t>(w, h, 0);
        std::uniform_int_distribution<int> dd(0, 255), vv(0, 3);
        for (int i = 0; i < w * h; ++i) {
            dm.d.data()[i] = dd(rng);
            dm.valid.data()[i] = vv(rng) != 0 && dm.d.data()[i] > 0;
        }
        tsgm::write_disparity_png(tmp + "/m.png", dm);
        const std::string p = "map_" + std::to_string(c);
        rec(p + "__d", "i4", {static_cast<uint32_t>(h), static_cast<uint32_t>(w)}, dm.d.data(),
            4 * static_cast<size_t>(w) * h);
        rec(p + "__valid", "u1", {static_cast<uint32_t>(h), static_cast<uint32_t>(w)},
            dm.valid.data(), static_cast<size_t>(w) * h);
        rec(p + "__raw", "u2", {static_cast<uint32_t>(h), static_cast<uint32_t>(w)},
            tsgm_shim::last16.data(), 2 * static_cast<size_t>(w) * h);
    }
    // values the 16-bit format cannot hold: the reference's error message
    const double bad[] = {256.0, -3.5, 0.001, 300.25};
    for (int c = 0; c < 4; ++c) {
        tsgm::Image<double> disp(9, 7, 1.0);
        disp(4, 5) = bad[c];
        std::string msg = "ok";
        try {
            tsgm::write_disparity_png(tmp + "/e.png", disp);
        } catch (const std::invalid_argument& e) {
            msg = e.what();
        }
        const std::string p = "bad_" + std::to_string(c);
        rec(p + "__disp", "f8", {7u, 9u}, disp.data(), 8 * 63);
        rec_text(p + "__msg", msg);
    }
    // boxes.txt
    {
        std::vector<std::vector<tsgm::DetectionBox>> per_frame(5);
        std::uniform_int_distribution<int> nb(0, 4), xy(0, 1200);
        std::uniform_real_distribution<double> sc(0.0, 40.0);
        std::vector<double> flat;
        std::vector<int32_t> counts;
        for (auto& f : per_frame) {
            const int n = nb(rng);
            for (int i = 0; i < n; ++i) {
                tsgm::DetectionBox bx;
                bx.x0 = xy(rng);
                bx.y0 = xy(rng) % 370;
                bx.x1 = bx.x0 + 20 + xy(rng) % 50;
                bx.y1 = bx.y0 + 20 + xy(rng) % 50;
                bx.score = sc(rng);
                if (i == 1) bx.score = 1.0 / 3.0;  // 17 significant digits
                f.push_back(bx);
                flat.insert(flat.end(), {double(bx.x0), double(bx.y0), double(bx.x1), double(bx.y1),
                                         bx.score});
            }
            counts.push_back(n);
        }
        tsgm::write_boxes(tmp + "/boxes.txt", per_frame);
        std::ifstream in(tmp + "/boxes.txt");
        std::stringstream ss;
        ss << in.rdbuf();
        rec("boxes__flat", "f8", {static_cast<uint32_t>(flat.size() / 5), 5u}, flat.data(),
            8 * flat.size());
        rec("boxes__counts", "i4", {static_cast<uint32_t>(counts.size())}, counts.data(),
            4 * counts.size());
        rec_text("boxes__text", ss.str());
    }
    std::fclose(g_out);
    return 0;
}
