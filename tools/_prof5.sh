bash tools/_tr5.sh
bash tools/_prof4.sh
