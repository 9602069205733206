// `ttswe` command-line tool of the B200 build (reference: proj/tools/ttswe_main.cpp:1-3).
#include "harness.hpp"

int main(int argc, char** argv) { return ttswe::run_cli(argc, argv); }
