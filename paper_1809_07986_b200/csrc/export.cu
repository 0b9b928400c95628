// Export formats: the reference's KITTI-style 16-bit
// disparity PNG (write_disparity_png, dataset.cpp:229-254: round(256·d), 0 =
// invalid) and boxes.txt (write_boxes, dataset.cpp:256-269).
//
// The quantisation runs on the device next to the maps it reads (the export
// map never leaves HBM as i32 + u8: 2 B/px cross PCIe instead of 5); the
// reference's per-pixel test is kept exactly — d == 0 is invalid, else
// v = lround(d·256) as a 64-bit long and 0 < v <= 65535 or the call fails
// with the reference's message at the FIRST such pixel in raster order (an
// atomicMin over the linear index). The container format is host work: a
// 16-bit grayscale PNG (IHDR, one zlib IDAT, IEND; filter type 0 per row).
// libpng is not in this image, so the bytes are not libpng's; the decoded
// pixels are the reference's (tests decode them).
#include <zlib.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace tsgm {

__global__ void quantize_disparity_kernel(const double* disp, const int32_t* d, const uint8_t* valid,
                                          size_t P, const int* slots, uint16_t* raw,
                                          unsigned long long* first_bad) {
    const int a = blockIdx.y;
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i >= P) return;
    const size_t src = static_cast<size_t>(slots ? slots[a] : a) * P + i;
    // write_disparity_png(DisparityMap): valid -> double(d), else 0 (dataset.cpp:247-253)
    const double v = disp ? disp[src] : (valid[src] ? static_cast<double>(d[src]) : 0.0);
    uint16_t out = 0;
    if (v != 0.0) {
        const long long q = x86_lround_long(__dmul_rn(v, 256.0));
        if (q <= 0 || q > 65535)
            atomicMin(first_bad + a, static_cast<unsigned long long>(i));
        else
            out = static_cast<uint16_t>(q);
    }
    raw[static_cast<size_t>(a) * P + i] = out;
}

void launch_quantize_disparity(const double* disp, const int32_t* d, const uint8_t* valid,
                               size_t P, int n, const int* slots, uint16_t* raw,
                               unsigned long long* first_bad, Launch L) {
    cudaMemsetAsync(first_bad, 0xff, sizeof(unsigned long long) * n, L.st);  // (checked by the caller's sync)
    quantize_disparity_kernel<<<dim3(static_cast<unsigned>((P + 255) / 256), n), 256, 0, L.st>>>(
        disp, d, valid, P, slots, raw, first_bad);
    ++*L.counter;
}

namespace {

void put_be32(std::vector<uint8_t>& v, uint32_t x) {
    v.push_back(static_cast<uint8_t>(x >> 24));
    v.push_back(static_cast<uint8_t>(x >> 16));
    v.push_back(static_cast<uint8_t>(x >> 8));
    v.push_back(static_cast<uint8_t>(x));
}

void put_chunk(std::vector<uint8_t>& png, const char* type, const uint8_t* data, size_t n) {
    put_be32(png, static_cast<uint32_t>(n));
    const size_t start = png.size();
    png.insert(png.end(), type, type + 4);
    if (n) png.insert(png.end(), data, data + n);
    const uLong crc = crc32(0L, png.data() + start, static_cast<uInt>(4 + n));
    put_be32(png, static_cast<uint32_t>(crc));
}

}  // namespace

void write_png16(const std::string& path, const uint16_t* raw, int w, int h) {
    // rows: filter byte 0, then big-endian samples
    const size_t row = 1 + 2 * static_cast<size_t>(w);
    std::vector<uint8_t> filt(row * static_cast<size_t>(h));
    for (int y = 0; y < h; ++y) {
        uint8_t* r = filt.data() + row * y;
        r[0] = 0;
        const uint16_t* s = raw + static_cast<size_t>(y) * w;
        for (int x = 0; x < w; ++x) {
            r[1 + 2 * x] = static_cast<uint8_t>(s[x] >> 8);
            r[2 + 2 * x] = static_cast<uint8_t>(s[x]);
        }
    }
    uLongf zlen = compressBound(static_cast<uLong>(filt.size()));
    std::vector<uint8_t> z(zlen);
    // level 1: 3-4x faster than libpng's default level 6 for a few % larger files
    if (compress2(z.data(), &zlen, filt.data(), static_cast<uLong>(filt.size()), 1) != Z_OK)
        throw std::runtime_error(path + ": PNG encode error");
    std::vector<uint8_t> png = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
    std::vector<uint8_t> ihdr;
    put_be32(ihdr, static_cast<uint32_t>(w));
    put_be32(ihdr, static_cast<uint32_t>(h));
    ihdr.insert(ihdr.end(), {16, 0, 0, 0, 0});  // 16-bit, grayscale, deflate, filter 0, no interlace
    put_chunk(png, "IHDR", ihdr.data(), ihdr.size());
    put_chunk(png, "IDAT", z.data(), zlen);
    put_chunk(png, "IEND", nullptr, 0);
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "wb"), &std::fclose);
    if (!f) throw std::runtime_error("cannot open file: " + path);  // image_io.cpp:25-29
    if (std::fwrite(png.data(), 1, png.size(), f.get()) != png.size())
        throw std::runtime_error(path + ": PNG encode error");
}

}  // namespace tsgm
