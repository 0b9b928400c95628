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
#include <cstdlib>
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

// read_disparity_png's decode (dataset.cpp:220-227 via image_io.cpp:172-193):
// a 16-bit single-channel, non-interlaced PNG, any of the five row filters,
// IDAT chunks concatenated and inflated with zlib. w/h out; raw resized.
void read_png16(const std::string& path, std::vector<uint16_t>& raw, int& w, int& h) {
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
    if (!f) throw std::runtime_error("cannot open file: " + path);
    std::vector<uint8_t> data;
    uint8_t buf[65536];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f.get())) > 0) data.insert(data.end(), buf, buf + n);
    static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
    if (data.size() < 8 || std::memcmp(data.data(), sig, 8) != 0)
        throw std::runtime_error(path + ": unsupported image format (expected PGM or PNG)");
    auto be32 = [&](size_t i) {
        return (uint32_t(data[i]) << 24) | (uint32_t(data[i + 1]) << 16) | (uint32_t(data[i + 2]) << 8) |
               uint32_t(data[i + 3]);
    };
    std::vector<uint8_t> idat;
    bool have_hdr = false;
    int depth = 0, color = 0, interlace = 0;
    for (size_t i = 8; i + 8 <= data.size();) {
        const uint32_t len = be32(i);
        if (i + 12 + len > data.size()) throw std::runtime_error(path + ": PNG decode error");
        const uint8_t* type = data.data() + i + 4;
        const uint8_t* body = data.data() + i + 8;
        // every chunk's CRC-32 over type + data, as libpng checks it
        const uLong crc = crc32(crc32(0L, Z_NULL, 0), type, 4 + len);
        if (crc != be32(i + 8 + len)) throw std::runtime_error(path + ": PNG decode error");
        if (!std::memcmp(type, "IHDR", 4) && len >= 13) {
            w = static_cast<int>(be32(i + 8));
            h = static_cast<int>(be32(i + 12));
            depth = body[8];
            color = body[9];
            interlace = body[12];
            have_hdr = true;
        } else if (!std::memcmp(type, "IDAT", 4)) {
            idat.insert(idat.end(), body, body + len);
        } else if (!std::memcmp(type, "IEND", 4)) {
            break;
        }
        i += 12 + len;
    }
    if (!have_hdr || depth != 16 || color != 0 || interlace != 0 || w <= 0 || h <= 0)
        throw std::runtime_error(path + ": expected 16-bit single-channel PNG");
    const size_t row = 2 * static_cast<size_t>(w);
    std::vector<uint8_t> fl((row + 1) * static_cast<size_t>(h));
    uLongf got = static_cast<uLongf>(fl.size());
    if (uncompress(fl.data(), &got, idat.data(), static_cast<uLong>(idat.size())) != Z_OK ||
        got != fl.size())
        throw std::runtime_error(path + ": PNG decode error");
    std::vector<uint8_t> prev(row, 0), cur(row);
    raw.assign(static_cast<size_t>(w) * h, 0);
    for (int y = 0; y < h; ++y) {
        const uint8_t ft = fl[(row + 1) * y];
        const uint8_t* in = fl.data() + (row + 1) * y + 1;
        for (size_t x = 0; x < row; ++x) {
            const int a = x >= 2 ? cur[x - 2] : 0, b = prev[x], c = x >= 2 ? prev[x - 2] : 0;
            int pr = 0;
            switch (ft) {
                case 0: pr = 0; break;
                case 1: pr = a; break;
                case 2: pr = b; break;
                case 3: pr = (a + b) / 2; break;
                case 4: {
                    const int p = a + b - c, pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
                    pr = (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
                    break;
                }
                default: throw std::runtime_error(path + ": PNG decode error");
            }
            cur[x] = static_cast<uint8_t>(in[x] + pr);
        }
        for (int x = 0; x < w; ++x)
            raw[static_cast<size_t>(y) * w + x] = static_cast<uint16_t>((cur[2 * x] << 8) | cur[2 * x + 1]);
        std::swap(prev, cur);
    }
}

}  // namespace tsgm
