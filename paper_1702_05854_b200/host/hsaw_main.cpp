// Entry point of the `hsaw` binary (reference: proj/tools/hsaw_main.cpp).
#include <string>
#include <vector>

#include "hsaw_b200.hpp"

int main(int argc, char** argv) {
    return hsaw::run_cli(std::vector<std::string>(argv + (argc > 0 ? 1 : 0), argv + argc));
}
