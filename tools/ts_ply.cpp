// ts_ply — PLY conversion through tilesplat/ply.hpp (host only, no device):
//   ts_ply <in.ply> <out.ply> [binary|ascii]
// Reads a 3DGS-layout PLY into a ParameterStore and writes
// it back; used by the CPU tests to cross-check the C++ and Python codecs.
#include <cstdio>
#include <string>

#include "tilesplat/ply.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: ts_ply <in.ply> <out.ply> [binary|ascii]\n");
        return 1;
    }
    try {
        const tilesplat::ParameterStore s = tilesplat::ply::read(argv[1]);
        const bool binary = argc < 4 || std::string(argv[3]) != "ascii";
        tilesplat::ply::write(argv[2], s, binary);
        std::printf("{\"n\": %lld}\n", (long long)s.size());
        return 0;
    } catch (const tilesplat::Error& e) {
        std::fprintf(stderr, "ts_ply: %s\n", e.what());
        return 1;
    }
}
