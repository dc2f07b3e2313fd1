// npy_tool.cpp — the reference's .npy writer / reader (kittensim npy.hpp:18-87) as a
// command-line tool, so KAT fixtures are written and read in the reference's own on-disk
// format. TEST INFRASTRUCTURE ONLY (built into oracle/_ref/).
//   npy_tool save <raw float32 file> <out.npy> <dim0> [dim1 ...]
//   npy_tool load <in.npy> <raw float32 out file>      (prints the shape)
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "kittensim/npy.hpp"

int main(int argc, char** argv) {
    try {
        if (argc >= 5 && std::string(argv[1]) == "save") {
            std::vector<std::size_t> shape;
            std::size_t n = 1;
            for (int i = 4; i < argc; ++i) {
                shape.push_back(std::strtoull(argv[i], nullptr, 10));
                n *= shape.back();
            }
            std::vector<float> data(n);
            std::ifstream in(argv[2], std::ios::binary);
            in.read(reinterpret_cast<char*>(data.data()), (std::streamsize)(n * 4));
            if (!in) return 3;
            kittensim::save_npy_f32(argv[3], data, shape);
            return 0;
        }
        if (argc == 4 && std::string(argv[1]) == "load") {
            std::vector<std::size_t> shape;
            auto data = kittensim::load_npy_f32(argv[2], shape);
            std::ofstream out(argv[3], std::ios::binary);
            out.write(reinterpret_cast<const char*>(data.data()), (std::streamsize)(data.size() * 4));
            for (auto s : shape) std::printf("%zu ", s);
            std::printf("\n");
            return 0;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 2;
    }
    std::fprintf(stderr, "usage: npy_tool save|load ...\n");
    return 1;
}
